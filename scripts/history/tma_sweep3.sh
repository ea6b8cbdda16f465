#!/bin/bash
set -u
O=gpurun_out/tma5; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4 > $O/pytest.txt
for red in sum max; do
  timeout 300 python bench.py --config rmat --reduce $red --steps 10 --no-e2e --no-cpu --no-variants > $O/rmat_${red}.json 2>$O/rmat_${red}.err
  PYG_SEG_TMA=0 timeout 300 python bench.py --config rmat --reduce $red --steps 10 --no-e2e --no-cpu --no-variants > $O/rmat_${red}_ldg.json 2>$O/rmat_${red}_ldg.err
done
for cfg in pubmed clouds cora; do timeout 300 python bench.py --config $cfg --steps 50 --no-e2e --no-variants > $O/$cfg.json 2>$O/$cfg.err; done
timeout 300 python bench.py --steps 10 --no-e2e --no-cpu --no-variants > $O/reddit.json 2>$O/reddit.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_rmat_sum.csv python bench.py --config rmat --steps 1 --warmup 3 --no-e2e --no-cpu --no-variants > /dev/null 2>&1
