#!/bin/bash
# halo push host-ordered + peer flags; ncu --set full of the L2-tiled atomic kernel (Reddit mean)
O=gpurun_out/r3d; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_halo_push.py tests/test_gpu_bench_multi.py -q -x 2>&1 | tail -5 > $O/tests.txt
Q="--steps 1 --warmup 1 --no-e2e --no-cpu --no-variants"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:coo_kernel -s 1 -c 1 -o $O/full_reddit_mean_atomic python bench.py --strategy atomic $Q > /dev/null 2>&1
ncu -i $O/full_reddit_mean_atomic.ncu-rep --page raw --csv > $O/full_reddit_mean_atomic.raw.csv 2>/dev/null
ncu -i $O/full_reddit_mean_atomic.ncu-rep --page details --csv > $O/full_reddit_mean_atomic.details.csv 2>/dev/null
ncu -i $O/full_reddit_mean_atomic.ncu-rep --page source --csv > $O/full_reddit_mean_atomic.source.csv 2>/dev/null
rm -f $O/*.ncu-rep
