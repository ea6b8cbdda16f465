#!/bin/bash
# GAT training step with the forward on a source-blocked plan when z exceeds L2
O=gpurun_out/r3ac; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_attention.py -q 2>&1 | tail -3 > $O/tests.txt
timeout 900 python bench.py --config reddit --op gat --steps 5 --no-e2e > $O/bench_gat_reddit.json 2> $O/bench_gat_reddit.err
timeout 900 python bench.py --config rmat --op gat --steps 5 --no-e2e > $O/bench_gat_rmat.json 2> $O/bench_gat_rmat.err
timeout 300 python bench.py --config pubmed --op gat --steps 20 --no-e2e > $O/bench_gat_pubmed.json 2> $O/bench_gat_pubmed.err
