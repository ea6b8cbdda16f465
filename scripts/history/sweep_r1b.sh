#!/bin/bash
set -u
mkdir -p gpurun_out/sweep2
for v in default minb2; do
  if [ "$v" = default ]; then unset PYG_LIBPATH; else export PYG_LIBPATH=$PWD/paper_1903_02428_b200/libpygs_$v.so; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-variants > gpurun_out/sweep2/reddit_${v}.json 2> gpurun_out/sweep2/reddit_${v}.err
  for red in sum max; do
    timeout 600 python bench.py --config rmat --reduce $red --steps 5 --warmup 3 --no-e2e --no-cpu --no-variants \
      > gpurun_out/sweep2/rmat_${red}_${v}.json 2> gpurun_out/sweep2/rmat_${red}_${v}.err
  done
done
unset PYG_LIBPATH
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sweep2/launches_rmat_sum.csv \
  python bench.py --config rmat --reduce sum --steps 2 --warmup 3 --no-e2e --no-cpu --no-variants > /dev/null 2>&1
