# round 2: the C-ABI multi-GPU layer (world 1 NCCL), the two-rank forward+backward vs oracle,
# bench's capi path, and the atomic R-MAT launch list
python -m pytest tests/test_gpu_dist.py tests/test_gpu_dist_backward.py tests/test_gpu_bench_multi.py tests/test_gpu_parity.py -q -x 2>&1 | tail -30 > gpurun_out/r2c_tests.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2c_launches_rmat_atomic_sum.csv python bench.py --config rmat --strategy atomic --reduce sum --steps 1 --warmup 3 --no-cpu --no-e2e --no-variants > /dev/null 2>&1
