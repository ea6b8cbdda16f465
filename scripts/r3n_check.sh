#!/bin/bash
# pipelined e2e (double-buffered inputs): default line + atomic mean line with e2e
O=gpurun_out/r3n; mkdir -p $O
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --config rmat --reduce sum --steps 5 --no-cpu --no-variants > $O/bench_rmat_sum.json 2> $O/bench_rmat_sum.err
timeout 600 python bench.py --strategy atomic --steps 5 --no-cpu --no-variants > $O/bench_reddit_atomic.json 2> $O/bench_reddit_atomic.err
