#!/bin/bash
# atomic lines with the bench's sampled oracle check (the tile kernel and compact tiles at full size)
O=gpurun_out/r3ab; mkdir -p $O
for red in mean max sum; do
  timeout 900 python bench.py --strategy atomic --reduce $red --steps 5 --no-variants --no-e2e > $O/bench_reddit_${red}_atomic.json 2> $O/bench_reddit_${red}_atomic.err
done
timeout 900 python bench.py --config rmat --reduce sum --strategy atomic --steps 5 --no-variants --no-e2e > $O/bench_rmat_sum_atomic.json 2> $O/bench_rmat_sum_atomic.err
for cfg in pubmed clouds cora; do
  timeout 300 python bench.py --config $cfg --strategy atomic --steps 50 --no-e2e --no-variants > $O/bench_${cfg}_atomic.json 2> $O/bench_${cfg}_atomic.err
done
