#!/bin/bash
# source-block size around the default (11 passes) for Reddit mean / max
O=gpurun_out/r3ak; mkdir -p $O
for i in 1 2; do
for cb in 21179 23297 25885; do
  for red in mean max; do
    timeout 600 python bench.py --reduce $red --col-block $cb --steps 10 --no-e2e --no-cpu --no-variants > $O/${red}_cb${cb}_$i.json 2>/dev/null
  done
done
done
