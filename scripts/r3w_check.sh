#!/bin/bash
# final state: GPU suite, smoke, default bench line, reference arm, R-MAT lines with their CPU baseline
O=gpurun_out/r3w; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $O/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1; echo "exit=$?" >> $O/smoke.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
for red in sum max; do
  timeout 900 python bench.py --config rmat --reduce $red --steps 10 --no-variants > $O/bench_rmat_$red.json 2> $O/bench_rmat_$red.err
done
