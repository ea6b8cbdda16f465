#!/bin/bash
# MAX fast path + compaction span heuristic: parity + atomic lines + launch list
O=gpurun_out/r3l; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x -k "atomic or coo or scatter or backward or propagate_random or concat or config" 2>&1 | tail -3 > $O/tests.txt
Q="--steps 5 --no-e2e --no-cpu --no-variants"
for red in mean sum max; do
  timeout 600 python bench.py --strategy atomic --reduce $red $Q > $O/reddit_${red}_atomic.json 2>$O/reddit_${red}_atomic.err
done
PYG_COO_COMPACT=0 timeout 600 python bench.py --strategy atomic --reduce mean $Q > $O/reddit_mean_atomic_inplace.json 2>/dev/null
for cfg in pubmed clouds cora; do
  timeout 300 python bench.py --config $cfg --strategy atomic --steps 50 --no-e2e --no-variants --no-cpu > $O/${cfg}_atomic.json 2>/dev/null
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__inst_executed.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/launches_reddit_mean_atomic.csv python bench.py --strategy atomic --steps 1 --warmup 1 --no-e2e --no-cpu --no-variants > /dev/null 2>&1
gzip -f $O/launches_reddit_mean_atomic.csv
