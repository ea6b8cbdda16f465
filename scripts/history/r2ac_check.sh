# Reddit max: column tiles (PYG_MAX_TILES) with the narrow packed-argmax build (U = 2) vs the default
O=gpurun_out/r2ac; mkdir -p $O
L=$PWD/paper_1903_02428_b200
Q="--reduce max --steps 10 --no-cpu --no-e2e --no-variants"
for i in 1 2; do
  python bench.py $Q > $O/max_base_$i.json 2>/dev/null
  PYG_MAX_TILES=2 python bench.py $Q > $O/max_t2_$i.json 2>/dev/null
  PYG_LIBPATH=$L/libpygs_narrow.so PYG_MAX_TILES=2 python bench.py $Q > $O/max_narrow_t2_$i.json 2>/dev/null
  PYG_LIBPATH=$L/libpygs_narrow.so PYG_MAX_TILES=3 python bench.py $Q > $O/max_narrow_t3_$i.json 2>/dev/null
done
PYG_LIBPATH=$L/libpygs_narrow.so PYG_MAX_TILES=2 timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -k "blocked and max" 2>&1 | tail -2 > $O/tests_narrow_t2.log
