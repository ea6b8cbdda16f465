# A/B: Reddit max with U=1 / 3 CTAs per SM (libpygs_maxu1.so) vs the default; atomic hub bitmap
O=gpurun_out/r2e; mkdir -p $O
python -m pytest tests/test_gpu_configs.py -q -k "atomic or blocked" 2>&1 | tail -3 > $O/tests.log
for i in 1 2; do
  python bench.py --reduce max --steps 10 --no-cpu --no-e2e --no-variants > $O/max_new_$i.json 2>/dev/null
  PYG_LIBPATH=$PWD/paper_1903_02428_b200/libpygs_maxu1.so python bench.py --reduce max --steps 10 --no-cpu --no-e2e --no-variants > $O/max_u1_$i.json 2>/dev/null
done
PYG_LIBPATH=$PWD/paper_1903_02428_b200/libpygs_maxu1.so python -m pytest tests/test_gpu_configs.py -q -k "blocked and max" 2>&1 | tail -2 > $O/tests_u1.log
python bench.py --config rmat --strategy atomic --reduce sum --steps 5 --no-cpu --no-e2e --no-variants > $O/rmat_atomic_sum.json 2>/dev/null
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -k regex:"coo|degree|hub|zero_slots|mean_div|max_decode" --csv --log-file $O/launches_rmat_atomic_sum.csv python bench.py --config rmat --strategy atomic --reduce sum --steps 1 --warmup 3 --no-cpu --no-e2e --no-variants > /dev/null 2>&1
