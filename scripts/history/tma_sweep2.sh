#!/bin/bash
set -u
O=gpurun_out/tma4; mkdir -p $O
for cfg in "8 4" "8 6" "8 8" "8 10" "4 8" "16 8" "4 6" "2 8"; do
  set -- $cfg
  for red in sum max; do
  PYG_TMA_WARPS=$1 PYG_TMA_WARP_KB=$2 timeout 300 python bench.py --config rmat --reduce $red --steps 5 --no-e2e --no-cpu --no-variants > $O/rmat_${red}_w$1_kb$2.json 2>$O/rmat_${red}_w$1_kb$2.err
  done
done
# TMA on the other configs (pubmed F=500, clouds F=64, reddit unblocked F=602)
for kb in 8 12 20; do
  PYG_TMA_WARP_KB=$kb timeout 300 python bench.py --config reddit --col-block 0 --steps 5 --no-e2e --no-cpu --no-variants > $O/reddit_unblocked_kb$kb.json 2>$O/reddit_unblocked_kb$kb.err
  PYG_TMA_WARP_KB=$kb timeout 300 python bench.py --config pubmed --steps 50 --no-e2e --no-cpu --no-variants > $O/pubmed_kb$kb.json 2>$O/pubmed_kb$kb.err
done
PYG_SEG_TMA=0 timeout 300 python bench.py --config pubmed --steps 50 --no-e2e --no-cpu --no-variants > $O/pubmed_ldg.json 2>$O/pubmed_ldg.err
PYG_SEG_TMA=0 timeout 300 python bench.py --config reddit --col-block 0 --steps 5 --no-e2e --no-cpu --no-variants > $O/reddit_unblocked_ldg.json 2>$O/reddit_unblocked_ldg.err
