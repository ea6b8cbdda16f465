#!/bin/bash
# tile kernel distinct-target fast path: atomic parity + atomic lines
O=gpurun_out/r3h; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x -k "atomic or coo or scatter or backward or propagate_random or concat or config" 2>&1 | tail -3 > $O/tests.txt
Q="--steps 5 --no-e2e --no-cpu --no-variants"
for red in mean sum max; do
  timeout 600 python bench.py --strategy atomic --reduce $red $Q > $O/reddit_${red}_atomic.json 2>/dev/null
done
for cfg in pubmed clouds cora; do
  timeout 300 python bench.py --config $cfg --strategy atomic --steps 50 --no-e2e --no-variants --no-cpu > $O/${cfg}_atomic.json 2>/dev/null
done
timeout 600 python bench.py --config rmat --reduce sum --strategy atomic $Q > $O/rmat_sum_atomic.json 2>/dev/null
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_op_red.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:coo_ --csv --log-file $O/launches_reddit_mean_atomic.csv python bench.py --strategy atomic --steps 1 --warmup 1 --no-e2e --no-cpu --no-variants > /dev/null 2>&1
