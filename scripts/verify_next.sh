#!/bin/bash
# Verification run for the latest kernel changes: full GPU suite + the affected bench lines.
O=gpurun_out/${1:-v}
mkdir -p $O
timeout -s KILL 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $O/pytest.txt
for red in sum max; do
  for i in 1 2; do timeout 300 python bench.py --config rmat --reduce $red --steps 10 --no-e2e --no-cpu --no-variants > $O/rmat_${red}_$i.json 2>/dev/null; done
done
timeout 300 python bench.py --steps 10 --no-e2e --no-cpu > $O/reddit.json 2>/dev/null
