#!/bin/bash
# GAT backward with a source-blocked transposed plan (grad_out rows L2-resident per pass)
O=gpurun_out/r3an; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_attention.py -q 2>&1 | tail -3 > $O/tests.txt
timeout 900 python bench.py --config reddit --op gat --steps 5 --no-e2e > $O/bench_gat_reddit.json 2> $O/bench_gat_reddit.err
PYG_BENCH_GAT_BLOCKED_MAX_F=1024 timeout 900 python bench.py --config reddit --op gat --steps 5 --no-e2e --no-cpu > $O/bench_gat_reddit_fwdblocked.json 2> $O/bench_gat_reddit_fwdblocked.err
timeout 900 python bench.py --config rmat --op gat --steps 5 --no-e2e --no-cpu > $O/bench_gat_rmat.json 2> $O/bench_gat_rmat.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"gat_|seg_|softmax|combine" --csv --log-file $O/launches_gat_reddit.csv python bench.py --config reddit --op gat --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
