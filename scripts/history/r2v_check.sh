# seg_kernel A/B: packed 16-bit argmax (U = 1) and persistent grid-stride rows, Reddit mean / sum / max + GCN 512
O=gpurun_out/r2v; mkdir -p $O
L=$PWD/paper_1903_02428_b200
for i in 1 2; do
  for v in base pack pers1 pers2 packpers; do
    lib=$L/libpygs_$v.so; [ $v = base ] && lib=$L/libpygs.so
    PYG_LIBPATH=$lib python bench.py --reduce max --steps 10 --no-cpu --no-e2e --no-variants > $O/max_${v}_$i.json 2>/dev/null
    PYG_LIBPATH=$lib python bench.py --reduce mean --steps 10 --no-cpu --no-e2e --no-variants > $O/mean_${v}_$i.json 2>/dev/null
  done
done
for v in base pers1 pers2; do
  lib=$L/libpygs_$v.so; [ $v = base ] && lib=$L/libpygs.so
  PYG_LIBPATH=$lib python bench.py --reduce sum --steps 10 --no-cpu --no-e2e --no-variants > $O/sum_${v}.json 2>/dev/null
  PYG_LIBPATH=$lib python bench.py --op gcn --hidden 512 --steps 10 --no-cpu --no-e2e > $O/gcn512_${v}.json 2>/dev/null
  PYG_LIBPATH=$lib python bench.py --config pubmed --steps 20 --no-cpu --no-e2e > $O/pubmed_${v}.json 2>/dev/null
done
for v in pack packpers pers1; do
  PYG_LIBPATH=$L/libpygs_$v.so timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3 > $O/tests_$v.log
done
