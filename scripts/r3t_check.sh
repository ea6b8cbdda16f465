#!/bin/bash
# after the narrow-row V = 8 rule: GPU suite, smoke, small configs, Fig. 3
O=gpurun_out/r3t; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $O/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1; echo "exit=$?" >> $O/smoke.txt
for cfg in clouds cora pubmed; do
  timeout 300 python bench.py --config $cfg --steps 50 --no-e2e --no-variants > $O/bench_$cfg.json 2> $O/bench_$cfg.err
done
timeout 300 python bench.py --config clouds --op gat --steps 50 --no-e2e > $O/bench_gat_clouds.json 2>/dev/null
timeout 600 python bench.py --config reddit --op appnp --steps 5 > $O/bench_appnp_reddit.json 2> $O/bench_appnp_reddit.err
timeout 300 python bench.py --config pubmed --op appnp --steps 5 > $O/bench_appnp_pubmed.json 2> $O/bench_appnp_pubmed.err
timeout 600 python bench.py --config reddit --op gatlayer --steps 10 > $O/bench_gatlayer_reddit.json 2> $O/bench_gatlayer_reddit.err
timeout 600 python scripts/fig3.py --out $O/fig3.json > $O/fig3.log 2>&1
