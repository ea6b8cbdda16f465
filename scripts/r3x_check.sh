#!/bin/bash
# the bench's sampled oracle check for max (argmax mapped back to original edge ids)
O=gpurun_out/r3x; mkdir -p $O
timeout 900 python bench.py --config rmat --reduce max --steps 5 --no-variants --no-e2e > $O/bench_rmat_max.json 2> $O/bench_rmat_max.err
timeout 900 python bench.py --reduce max --steps 5 --no-variants --no-e2e > $O/bench_reddit_max.json 2> $O/bench_reddit_max.err
timeout 900 python bench.py --config clouds --steps 20 --no-variants --no-e2e > $O/bench_clouds.json 2> $O/bench_clouds.err
timeout 900 python bench.py --config rmat --reduce max --strategy atomic --steps 3 --no-variants --no-e2e > $O/bench_rmat_max_atomic.json 2> $O/bench_rmat_max_atomic.err
