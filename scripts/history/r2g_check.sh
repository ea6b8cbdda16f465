O=gpurun_out/r2g; mkdir -p $O
python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3 > $O/tests.log
python bench.py --reduce max --steps 10 --no-cpu --no-e2e --no-variants > $O/reddit_max.json 2>/dev/null
python bench.py --config rmat --reduce max --steps 10 --no-cpu --no-e2e --no-variants > $O/rmat_max.json 2>/dev/null
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -k regex:"seg_|combine|tf32|deg_rsqrt" --csv --log-file $O/launches_gcn512.csv python bench.py --op gcn --hidden 512 --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout 900 python scripts/cpu_full_pass.py reddit-mean rmat-sum > $O/cpu_full_pass.log 2>&1
cp profiles/cpu_full_pass.json $O/ 2>/dev/null
