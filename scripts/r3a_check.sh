#!/bin/bash
# session re-entry check: HEAD green on the GPU, default + max bench lines
O=gpurun_out/r3a; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > $O/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1; echo "exit=$?" >> $O/smoke.txt
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --reduce max --steps 10 --no-e2e --no-cpu --no-variants > $O/bench_reddit_max.json 2> $O/bench_reddit_max.err
timeout 600 python bench.py --config rmat --reduce max --strategy atomic --steps 5 --no-e2e --no-cpu --no-variants > $O/bench_rmat_max_atomic.json 2> $O/bench_rmat_max_atomic.err
timeout 600 python bench.py --strategy atomic --steps 5 --no-e2e --no-cpu --no-variants > $O/bench_reddit_mean_atomic.json 2> $O/bench_reddit_mean_atomic.err
