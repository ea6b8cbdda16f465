#!/bin/bash
# Verification run for the latest kernel changes: full GPU suite + the affected bench lines.
O=gpurun_out/${1:-v}
mkdir -p $O
timeout -s KILL 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $O/pytest.txt
for cfg in rmat pubmed; do timeout 400 python bench.py --config $cfg --op gat --steps 10 > $O/gat_$cfg.json 2>$O/gat_$cfg.err; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"softmax|seg_|combine|gat_" --csv --log-file $O/launches_gat_rmat.csv python bench.py --config rmat --op gat --steps 1 --no-cpu > /dev/null 2>&1
gzip -f $O/launches_gat_rmat.csv
for cfg in cora pubmed clouds; do timeout 300 python bench.py --config $cfg --steps 50 --no-e2e --no-variants > $O/$cfg.json 2>$O/$cfg.err; done
timeout 600 python scripts/fig3.py --out $O/fig3.json > $O/fig3.log 2>&1
