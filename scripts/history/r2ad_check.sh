# GAT forward: s_dst gathered per slot (no new-row tracking, no capture loop)
O=gpurun_out/r2ad; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_attention.py -q -x 2>&1 | tail -3 > $O/attention.log
for i in 1 2; do python bench.py --config rmat --op gat --steps 5 --no-cpu --no-e2e > $O/gat_rmat_$i.json 2>/dev/null; done
python bench.py --config rmat --op gatlayer --steps 10 --no-cpu --no-e2e > $O/gatlayer_rmat.json 2>/dev/null
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:"gat_" --csv --log-file $O/launches_gat_rmat.csv python bench.py --config rmat --op gat --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
