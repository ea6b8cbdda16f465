#!/bin/bash
# Reddit GAT training step at 8 x 64 (one-pass TMA forward and backward, blocked transposed plan)
O=gpurun_out/r3ao; mkdir -p $O
timeout 900 python bench.py --config reddit --op gat --steps 5 --no-e2e > $O/bench_gat_reddit.json 2> $O/bench_gat_reddit.err
PYG_BENCH_GAT_BLOCKED_MAX_F=1024 timeout 900 python bench.py --config reddit --op gat --steps 5 --no-e2e --no-cpu > $O/bench_gat_reddit_fwdblocked.json 2> $O/bench_gat_reddit_fwdblocked.err
timeout 900 python bench.py --config reddit --op gat --col-block 0 --steps 5 --no-e2e --no-cpu > $O/bench_gat_reddit_unblocked.json 2> $O/bench_gat_reddit_unblocked.err
