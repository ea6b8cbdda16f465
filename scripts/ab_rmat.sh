#!/bin/bash
# A/B of the R-MAT sum/max bench between the current tree and an older build in abtest/<tag>
set -u
O=gpurun_out/ab; mkdir -p $O
for i in 1 2; do
for red in sum max; do
  timeout 300 python bench.py --config rmat --reduce $red --steps 10 --no-e2e --no-cpu --no-variants > $O/new_${red}_$i.json 2>/dev/null
  (cd abtest/r1c && timeout 300 python bench.py --config rmat --reduce $red --steps 10 --no-e2e --no-cpu --no-variants > ../../$O/old_${red}_$i.json 2>/dev/null)
done
done
