#!/bin/bash
# warp-batched coo_tile_kernel: parity of every atomic-path test + A/B against the generic coo_kernel
O=gpurun_out/r3e; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x -k "atomic or coo or scatter or backward or propagate_random or concat or config or fig3 or appnp or gcn" 2>&1 | tail -15 > $O/tests.txt
Q="--steps 5 --no-e2e --no-cpu --no-variants"
for tile in 1 0; do
  for red in mean max; do
    PYG_COO_TILE=$tile timeout 600 python bench.py --strategy atomic --reduce $red $Q > $O/reddit_${red}_atomic_t$tile.json 2> $O/reddit_${red}_atomic_t$tile.err
  done
  for red in sum max; do
    PYG_COO_TILE=$tile timeout 600 python bench.py --config rmat --reduce $red --strategy atomic $Q > $O/rmat_${red}_atomic_t$tile.json 2> $O/rmat_${red}_atomic_t$tile.err
  done
  for cfg in pubmed clouds cora; do
    PYG_COO_TILE=$tile timeout 300 python bench.py --config $cfg --strategy atomic --steps 50 --no-e2e --no-variants --no-cpu > $O/${cfg}_atomic_t$tile.json 2> $O/${cfg}_atomic_t$tile.err
  done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
timeout 600 ncu --metrics $M --clock-control none -k regex:coo_ --csv --log-file $O/launches_reddit_mean_atomic.csv python bench.py --strategy atomic --steps 1 --warmup 1 --no-e2e --no-cpu --no-variants > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:coo_ --csv --log-file $O/launches_rmat_sum_atomic.csv python bench.py --config rmat --strategy atomic --reduce sum --steps 1 --warmup 1 --no-e2e --no-cpu --no-variants > /dev/null 2>&1
