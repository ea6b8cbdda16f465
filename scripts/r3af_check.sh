#!/bin/bash
# Reddit max: the row's packed keys prefetched into L2 at row start (libpygs.so) vs not (libpygs_old.so)
O=gpurun_out/r3af; mkdir -p $O
OLD=$PWD/paper_1903_02428_b200/libpygs_old.so
Q="--reduce max --steps 10 --no-e2e --no-cpu --no-variants"
for i in 1 2; do
  timeout 300 python bench.py $Q > $O/new_$i.json 2>/dev/null
  PYG_LIBPATH=$OLD timeout 300 python bench.py $Q > $O/old_$i.json 2>/dev/null
done
timeout 600 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -x -k "max or blocked or source" 2>&1 | tail -2 > $O/tests.txt
