#!/bin/bash
# Quick regression run: parity tests + the headline bench lines (results in gpurun_out/$1/).
set -u
O=gpurun_out/${1:-reg}
mkdir -p $O
timeout -s KILL 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > $O/pytest.txt
timeout 300 python bench.py --steps 10 --no-e2e --no-cpu --no-variants > $O/reddit_mean.json 2>/dev/null
for red in sum max; do
  timeout 300 python bench.py --config rmat --reduce $red --steps 10 --no-e2e --no-cpu --no-variants > $O/rmat_$red.json 2>/dev/null
done
