#!/bin/bash
O=gpurun_out/r3aq; mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"gat_|seg_|softmax|combine|scale_rows" --csv --log-file $O/launches_gat_reddit.csv python bench.py --config reddit --op gat --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
gzip -f $O/launches_gat_reddit.csv
