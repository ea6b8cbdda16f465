#!/bin/bash
# Round-1 tuning sweep: library variants x source-block sizes on the Reddit mean workload,
# plus the R-MAT configurations.  Results land in gpurun_out/sweep/.
set -u
mkdir -p gpurun_out/sweep
for v in default minb2 minb3; do
  if [ "$v" = default ]; then unset PYG_LIBPATH; else export PYG_LIBPATH=$PWD/paper_1903_02428_b200/libpygs_$v.so; fi
  for cb in 0 20000 30000 auto; do
    timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-variants --col-block $cb \
      > gpurun_out/sweep/reddit_${v}_$cb.json 2> gpurun_out/sweep/reddit_${v}_$cb.err
  done
done
unset PYG_LIBPATH
for red in sum max; do
  for st in segment atomic; do
    timeout 600 python bench.py --config rmat --reduce $red --strategy $st --steps 5 --warmup 3 --no-e2e --no-cpu --no-variants \
      > gpurun_out/sweep/rmat_${red}_$st.json 2> gpurun_out/sweep/rmat_${red}_$st.err
  done
done
