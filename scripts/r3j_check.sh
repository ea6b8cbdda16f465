#!/bin/bash
O=gpurun_out/r3j; mkdir -p $O
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/l2red scripts/l2red.cu && timeout 300 /tmp/l2red > $O/l2red.json 2> $O/l2red.err
