#!/bin/bash
O=gpurun_out/r3ap; mkdir -p $O
timeout 900 python bench.py --config reddit --op gat --steps 5 --no-e2e > $O/bench_gat_reddit.json 2> $O/bench_gat_reddit.err
timeout 900 python bench.py --config rmat --op gat --steps 5 --no-e2e > $O/bench_gat_rmat.json 2> $O/bench_gat_rmat.err
timeout 300 python bench.py --config pubmed --op gat --steps 20 --no-e2e > $O/bench_gat_pubmed.json 2> $O/bench_gat_pubmed.err
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $O/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1; echo "exit=$?" >> $O/smoke.txt
