#!/bin/bash
# ncu captures for the R-MAT configuration (segment sum light kernel, atomic sum kernel)
set -u
mkdir -p gpurun_out/rmat
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_kernel -s 3 -c 1 -o gpurun_out/rmat/prof_rmat_seg_sum \
  python bench.py --config rmat --reduce sum --steps 1 --warmup 3 --no-e2e --no-cpu --no-variants > gpurun_out/rmat/ncu_seg.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:coo_kernel -s 3 -c 1 -o gpurun_out/rmat/prof_rmat_coo_sum \
  python bench.py --config rmat --reduce sum --strategy atomic --steps 1 --warmup 3 --no-e2e --no-cpu --no-variants > gpurun_out/rmat/ncu_coo.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rmat/launches_rmat_seg_sum.csv \
  python bench.py --config rmat --reduce sum --steps 2 --warmup 3 --no-e2e --no-cpu --no-variants > /dev/null 2>&1
export PYG_LIBPATH=$PWD/paper_1903_02428_b200/libpygs_minb3.so
for red in sum max; do
  timeout 600 python bench.py --config rmat --reduce $red --steps 5 --warmup 3 --no-e2e --no-cpu --no-variants \
    > gpurun_out/rmat/rmat_${red}_minb3.json 2> gpurun_out/rmat/rmat_${red}_minb3.err
done
