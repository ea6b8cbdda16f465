#!/bin/bash
# R-MAT TMA ring / warps sweep for sum and max (env overrides of segment_tma.cu)
O=gpurun_out/${1:-tsw}; mkdir -p $O
for red in max sum; do
  for kb in 4 6 8; do
    for w in 4 8; do
      PYG_TMA_WARP_KB=$kb PYG_TMA_WARPS=$w timeout 300 python bench.py --config rmat --reduce $red --steps 10 --no-e2e --no-cpu --no-variants > $O/${red}_kb${kb}_w$w.json 2>/dev/null
    done
  done
done
