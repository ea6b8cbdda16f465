# round 2: L2 gather peak, Reddit blocked MAX with packed keys across passes, atomic R-MAT launch list
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/l2peak scripts/l2peak.cu && /tmp/l2peak > gpurun_out/r2d_l2peak.json 2>&1
python -m pytest tests/test_gpu_configs.py -q -k "blocked" 2>&1 | tail -5 > gpurun_out/r2d_tests.log
python bench.py --reduce max --steps 10 --no-cpu --no-e2e --no-variants > gpurun_out/r2d_reddit_max.json 2>gpurun_out/r2d_reddit_max.err
python bench.py --reduce mean --steps 10 --no-cpu --no-e2e > gpurun_out/r2d_reddit_mean.json 2>gpurun_out/r2d_reddit_mean.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -k regex:"coo|degree|hub|zero_slots|mean_div|max_decode" --csv --log-file gpurun_out/r2d_launches_rmat_atomic_sum.csv python bench.py --config rmat --strategy atomic --reduce sum --steps 1 --warmup 3 --no-cpu --no-e2e --no-variants > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:"seg_|combine" --csv --log-file gpurun_out/r2d_launches_reddit_max.csv python bench.py --reduce max --steps 1 --warmup 3 --no-cpu --no-e2e --no-variants > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:seg_kernel -s 40 -c 1 -o gpurun_out/r2d_full_reddit_max python bench.py --reduce max --steps 1 --warmup 3 --no-cpu --no-e2e --no-variants > /dev/null 2>&1
ncu -i gpurun_out/r2d_full_reddit_max.ncu-rep --page raw --csv > gpurun_out/r2d_full_reddit_max.raw.csv 2>/dev/null
ncu -i gpurun_out/r2d_full_reddit_max.ncu-rep --page details --csv > gpurun_out/r2d_full_reddit_max.details.csv 2>/dev/null
rm -f gpurun_out/r2d_full_reddit_max.ncu-rep
