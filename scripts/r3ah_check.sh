#!/bin/bash
# degree pass zeroes the in-place atomic target (one launch fewer per call)
O=gpurun_out/r3ah; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x -k "atomic or coo or scatter or backward or propagate or concat or config or dist or gcn or appnp" 2>&1 | tail -3 > $O/tests.txt
timeout 300 python bench.py --config cora --strategy atomic --steps 50 --no-e2e --no-variants > $O/cora_atomic.json 2>/dev/null
timeout 900 python bench.py --config rmat --reduce sum --strategy atomic --steps 5 --no-e2e --no-variants > $O/rmat_sum_atomic.json 2>/dev/null
timeout 900 python bench.py --strategy atomic --steps 5 --no-e2e --no-variants > $O/reddit_mean_atomic.json 2>/dev/null
timeout 600 python scripts/fig3.py --out $O/fig3.json > $O/fig3.log 2>&1
