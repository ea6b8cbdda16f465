#!/bin/bash
# e2e: next step's H2D enqueued before the host-synchronous plan build
O=gpurun_out/r3ag; mkdir -p $O
timeout 900 python bench.py --no-variants --no-cpu > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --strategy atomic --no-variants --no-cpu > $O/bench_atomic.json 2> $O/bench_atomic.err
timeout 900 python bench.py --config rmat --no-variants --no-cpu > $O/bench_rmat.json 2> $O/bench_rmat.err
