#!/bin/bash
# GAT: float4 chunks never straddle heads (C % 4 == 0 for the one-pass / blocked kernels)
O=gpurun_out/r3aa; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_attention.py -q 2>&1 | tail -3 > $O/tests.txt
timeout 600 python scripts/gat_reddit_check.py 2000 75 > $O/c75.txt 2>&1
timeout 600 python scripts/gat_reddit_check.py 2000 72 > $O/c72.txt 2>&1
timeout 900 python bench.py --config reddit --op gat --steps 5 --no-e2e > $O/bench_gat_reddit.json 2> $O/bench_gat_reddit.err
timeout 900 python bench.py --config rmat --op gat --steps 5 --no-e2e > $O/bench_gat_rmat.json 2> $O/bench_gat_rmat.err
