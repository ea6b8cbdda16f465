#!/bin/bash
# blocked GAT forward for wide rows (fewer z rows in flight, 2 CTAs / SM): Reddit GAT training step
O=gpurun_out/r3ad; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_attention.py -q 2>&1 | tail -3 > $O/tests.txt
PYG_BENCH_GAT_BLOCKED_MAX_F=1024 timeout 900 python bench.py --config reddit --op gat --steps 5 --no-e2e > $O/bench_gat_reddit_blocked.json 2> $O/bench_gat_reddit_blocked.err
timeout 900 python bench.py --config reddit --op gat --steps 5 --no-e2e --no-cpu > $O/bench_gat_reddit.json 2> $O/bench_gat_reddit.err
timeout 900 python bench.py --config reddit --op gatlayer --steps 10 --no-e2e > $O/bench_gatlayer_reddit.json 2> $O/bench_gatlayer_reddit.err
