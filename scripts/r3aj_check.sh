#!/bin/bash
# end-of-session state: GPU suite, smoke, default bench line
O=gpurun_out/r3aj; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $O/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1; echo "exit=$?" >> $O/smoke.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
