#!/bin/bash
# tile kernel: L2 budget and chunk sweep (Reddit mean / max, PubMed), clouds atomic line
O=gpurun_out/r3f; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "atomic or coo or scatter_random" 2>&1 | tail -3 > $O/tests.txt
Q="--steps 5 --no-e2e --no-cpu --no-variants"
for mb in 48 72 96 110; do
  for red in mean max; do
    PYG_COO_L2_MB=$mb timeout 600 python bench.py --strategy atomic --reduce $red $Q > $O/reddit_${red}_mb$mb.json 2>/dev/null
  done
  PYG_COO_L2_MB=$mb timeout 300 python bench.py --config pubmed --strategy atomic --steps 50 --no-e2e --no-variants --no-cpu > $O/pubmed_mb$mb.json 2>/dev/null
done
for ch in 128 512 2048; do
  PYG_COO_CHUNK=$ch timeout 600 python bench.py --strategy atomic --reduce mean $Q > $O/reddit_mean_ch$ch.json 2>/dev/null
done
timeout 300 python bench.py --config clouds --strategy atomic --steps 50 --no-e2e --no-variants --no-cpu > $O/clouds_atomic.json 2> $O/clouds_atomic.err
