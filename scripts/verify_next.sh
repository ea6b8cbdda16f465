#!/bin/bash
# Verification run for the latest kernel changes: full GPU suite + the affected bench lines.
O=gpurun_out/${1:-v}
mkdir -p $O
timeout -s KILL 1000 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $O/pytest.txt
timeout 600 python scripts/fig3.py --out $O/fig3.json > $O/fig3.log 2>&1
for cfg in cora pubmed clouds; do timeout 300 python bench.py --config $cfg --steps 50 --no-e2e --no-variants > $O/$cfg.json 2>/dev/null; done
for red in sum max; do timeout 300 python bench.py --config rmat --reduce $red --steps 10 --no-e2e --no-cpu --no-variants > $O/rmat_$red.json 2>/dev/null; done
