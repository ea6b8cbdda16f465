#!/bin/bash
# streamed alpha stores (__stcs) in the GAT forwards: libpygs.so vs PYG_GAT_STCS=0 (libpygs_old.so);
# GAT layer on Reddit at 5 (auto) and 8 passes, GAT fwd+bwd on R-MAT; plus the LDG vector-width test
O=gpurun_out/r3s; mkdir -p $O
OLD=$PWD/paper_1903_02428_b200/libpygs_old.so
for i in 1 2; do
  for cb in auto 29121; do
    timeout 600 python bench.py --config reddit --op gatlayer --col-block $cb --steps 10 --no-cpu --no-e2e > $O/gatl_cb${cb}_new_$i.json 2>/dev/null
    PYG_LIBPATH=$OLD timeout 600 python bench.py --config reddit --op gatlayer --col-block $cb --steps 10 --no-cpu --no-e2e > $O/gatl_cb${cb}_old_$i.json 2>/dev/null
  done
  timeout 600 python bench.py --config rmat --op gat --steps 5 --no-cpu --no-e2e > $O/gat_rmat_new_$i.json 2>/dev/null
  PYG_LIBPATH=$OLD timeout 600 python bench.py --config rmat --op gat --steps 5 --no-cpu --no-e2e > $O/gat_rmat_old_$i.json 2>/dev/null
done
timeout 900 python -m pytest tests/test_gpu_attention.py -q -x 2>&1 | tail -2 > $O/tests.txt
bash scripts/r3r_check.sh
# APPNP with the weights gathered into plan order once per call (r3p: Reddit 185.1 ms, PubMed 0.461 ms)
timeout 600 python bench.py --config reddit --op appnp --steps 5 > $O/appnp_reddit.json 2>/dev/null
timeout 600 python bench.py --config pubmed --op appnp --steps 5 > $O/appnp_pubmed.json 2>/dev/null
PYG_LIBPATH=$OLD timeout 600 python bench.py --config reddit --op appnp --steps 5 > $O/appnp_reddit_old.json 2>/dev/null
timeout 600 python -m pytest tests/test_gpu_appnp.py -q -x 2>&1 | tail -2 > $O/tests_appnp.txt
