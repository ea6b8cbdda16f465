#!/bin/bash
# L2 atomic-reduction roof (scripts/l2red.cu) + the host-ordered halo push / peer flag tests
O=gpurun_out/r3c; mkdir -p $O
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/l2red scripts/l2red.cu && timeout 300 /tmp/l2red > $O/l2red.json 2> $O/l2red.err
timeout 900 python -m pytest tests/test_gpu_halo_push.py tests/test_gpu_bench_multi.py -q -x 2>&1 | tail -5 > $O/tests.txt
