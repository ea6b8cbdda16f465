# GAT attention in factored form (row_sums): no E x H normalisation pass in the training step
O=gpurun_out/r2s; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_attention.py -q -x 2>&1 | tail -25 > $O/attention.log
Q="--config rmat --op gat --steps 5 --no-cpu --no-e2e"
python bench.py $Q > $O/gat.json 2>$O/gat.err
python bench.py --config pubmed --op gat --steps 20 --no-cpu --no-e2e > $O/gat_pubmed.json 2>/dev/null
python bench.py --config rmat --op gatlayer --steps 5 --no-cpu --no-e2e > $O/gatlayer_rmat.json 2>/dev/null
python bench.py --config reddit --op gatlayer --steps 5 --no-cpu --no-e2e > $O/gatlayer_reddit.json 2>/dev/null
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:"softmax|gat_|seg_|combine" --csv --log-file $O/launches_gat_rmat.csv python bench.py $Q --steps 1 --warmup 2 > /dev/null 2>&1
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1
