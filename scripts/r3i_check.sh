#!/bin/bash
# tile kernel with the next batch's indices prefetched: parity + Reddit atomic chunk sweep
O=gpurun_out/r3i; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x -k "atomic or coo or scatter or backward or propagate_random or concat" 2>&1 | tail -3 > $O/tests.txt
Q="--steps 5 --no-e2e --no-cpu --no-variants"
for ch in 128 512 2048; do
  PYG_COO_CHUNK=$ch timeout 600 python bench.py --strategy atomic --reduce mean $Q > $O/reddit_mean_ch$ch.json 2>/dev/null
done
timeout 600 python bench.py --strategy atomic --reduce max $Q > $O/reddit_max.json 2>/dev/null
for cfg in pubmed clouds cora; do
  timeout 300 python bench.py --config $cfg --strategy atomic --steps 50 --no-e2e --no-variants --no-cpu > $O/${cfg}_atomic.json 2>/dev/null
done
