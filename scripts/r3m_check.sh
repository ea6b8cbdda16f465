#!/bin/bash
# R-MAT atomic: tile kernel with fast paths (PYG_COO_TILE=2, 128-column rows) vs coo_kernel
O=gpurun_out/r3m; mkdir -p $O
Q="--steps 5 --no-e2e --no-cpu --no-variants"
for t in 1 2; do
  for red in sum max; do
    PYG_COO_TILE=$t timeout 600 python bench.py --config rmat --reduce $red --strategy atomic $Q > $O/rmat_${red}_t$t.json 2>/dev/null
  done
done
PYG_COO_TILE=2 timeout 900 python -m pytest tests -m gpu -q -x -k "atomic or coo or scatter_random or backward" 2>&1 | tail -3 > $O/tests_t2.txt
