#!/bin/bash
# atomic path with fewer launches per call (deg + counters in one memset, hubs zero their own slots)
O=gpurun_out/r3u; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x -k "atomic or coo or scatter or backward or propagate or concat or config or fig3 or dist" 2>&1 | tail -3 > $O/tests.txt
Q="--steps 5 --no-e2e --no-cpu --no-variants"
timeout 600 python bench.py --config rmat --reduce sum --strategy atomic $Q > $O/rmat_sum_atomic.json 2>/dev/null
timeout 600 python bench.py --strategy atomic $Q > $O/reddit_mean_atomic.json 2>/dev/null
timeout 300 python bench.py --config cora --strategy atomic --steps 50 --no-e2e --no-variants --no-cpu > $O/cora_atomic.json 2>/dev/null
timeout 600 python scripts/fig3.py --out $O/fig3.json > $O/fig3.log 2>&1
