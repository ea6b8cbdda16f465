#!/bin/bash
# Verification run for the latest kernel changes: full GPU suite + the affected bench lines.
O=gpurun_out/${1:-v}
mkdir -p $O
timeout -s KILL 1000 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $O/pytest.txt
timeout 300 python bench.py --steps 10 --no-e2e --no-cpu > $O/reddit.json 2>/dev/null
for op in appnp gcn; do timeout 400 python bench.py --config reddit --op $op --steps 5 --no-cpu > $O/reddit_$op.json 2>/dev/null; done
for op in gcn gat; do timeout 400 python bench.py --config rmat --op $op --steps 5 --no-cpu > $O/rmat_$op.json 2>/dev/null; done
