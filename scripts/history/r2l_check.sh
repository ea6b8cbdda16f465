# one-pass GAT backward (gat_tma.cu) parity + timing; bulk-kernel suite failure repro; Reddit max with bulk off
O=gpurun_out/r2l; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x 2>&1 | tail -30 > $O/attention.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -60 > $O/parity.log
python bench.py --config rmat --op gat --steps 5 --no-cpu --no-e2e > $O/gat_rmat.json 2>$O/gat_rmat.err
python bench.py --reduce max --steps 10 --no-cpu --no-e2e --no-variants > $O/reddit_max.json 2>/dev/null
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:"softmax|gat_|seg_|combine" --csv --log-file $O/launches_gat_rmat.csv python bench.py --config rmat --op gat --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1
