# Reddit max: argmax as packed 16-bit segment positions (PYG_MAX_PACK) with U edges in flight; A/B of builds
O=gpurun_out/r2u; mkdir -p $O
L=$PWD/paper_1903_02428_b200
Q="--reduce max --steps 10 --no-cpu --no-e2e --no-variants"
for i in 1 2; do
  python bench.py $Q > $O/max_base_$i.json 2>/dev/null
  for v in u1m3 u2m3 u2m2 u3m2; do PYG_LIBPATH=$L/libpygs_$v.so python bench.py $Q > $O/max_${v}_$i.json 2>/dev/null; done
done
for v in u2m2 u3m2; do
  PYG_LIBPATH=$L/libpygs_$v.so timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -x -k "max or blocked" 2>&1 | tail -3 > $O/tests_$v.log
done
