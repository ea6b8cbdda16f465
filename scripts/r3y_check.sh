#!/bin/bash
# Reddit GAT fwd + bwd (unblocked backward) and an ncu launch list of the GAT layer forward passes
O=gpurun_out/r3y; mkdir -p $O
timeout 900 python bench.py --config reddit --op gat --steps 5 --no-e2e > $O/bench_gat_reddit.json 2> $O/bench_gat_reddit.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed
timeout 900 ncu --metrics $M --clock-control none -k regex:"gat_|tf32" --csv --log-file $O/launches_gatlayer_reddit.csv python bench.py --config reddit --op gatlayer --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:"gat_|seg_|softmax|combine" --csv --log-file $O/launches_gat_reddit.csv python bench.py --config reddit --op gat --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
