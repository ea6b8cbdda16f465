#!/bin/bash
O=gpurun_out/r3ai; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x -k "atomic or coo or scatter or backward or propagate or concat" 2>&1 | tail -3 > $O/tests.txt
timeout 900 python bench.py --config rmat --reduce sum --strategy atomic --steps 5 --no-e2e --no-variants --no-cpu > $O/rmat_sum_atomic.json 2>/dev/null
timeout 300 python bench.py --config cora --strategy atomic --steps 50 --no-e2e --no-variants --no-cpu > $O/cora_atomic.json 2>/dev/null
