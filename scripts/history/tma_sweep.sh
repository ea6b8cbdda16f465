#!/bin/bash
set -u
O=gpurun_out/tma3; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tma or split or propagate_random" 2>&1 | tail -3 > $O/pytest.txt
for cfg in "8 12" "8 8" "16 6" "4 24" "16 4"; do
  set -- $cfg
  PYG_TMA_WARPS=$1 PYG_TMA_WARP_KB=$2 timeout 300 python bench.py --config rmat --reduce sum --steps 5 --no-e2e --no-cpu --no-variants > $O/rmat_sum_w$1_kb$2.json 2>$O/rmat_sum_w$1_kb$2.err
done
PYG_SEG_TMA=0 timeout 300 python bench.py --config rmat --reduce sum --steps 5 --no-e2e --no-cpu --no-variants > $O/rmat_sum_ldg.json 2>$O/rmat_sum_ldg.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --config rmat --steps 1 --warmup 3 --no-e2e --no-cpu --no-variants > /dev/null 2>&1
