# bulk-kernel failure diagnosis + Reddit max regression A/B (HEAD vs 449f460 build)
O=gpurun_out/r2k; mkdir -p $O
L=$PWD/paper_1903_02428_b200
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "bulk and 256-256" 2>&1 | grep -v "^$" | head -80 > $O/bulk_test.log
timeout 300 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -q -x -k "bulk and 256-256" > $O/bulk_sanitizer.log 2>&1
for i in 1 2; do
python bench.py --reduce max --steps 10 --no-cpu --no-e2e --no-variants > $O/max_head_$i.json 2>/dev/null
PYG_LIBPATH=$L/libpygs_449.so python bench.py --reduce max --steps 10 --no-cpu --no-e2e --no-variants > $O/max_449_$i.json 2>/dev/null
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/launches_max_head.csv python bench.py --reduce max --steps 1 --warmup 3 --no-e2e --no-cpu --no-variants > /dev/null 2>&1
PYG_LIBPATH=$L/libpygs_449.so timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/launches_max_449.csv python bench.py --reduce max --steps 1 --warmup 3 --no-e2e --no-cpu --no-variants > /dev/null 2>&1
