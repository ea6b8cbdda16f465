#!/bin/bash
# source-block size for narrow gathered rows: GCN 602 -> 128 on Reddit (H = 119 MB, unblocked by the
# current rule) and the GAT layer (z = 238 MB, 5 passes)
O=gpurun_out/r3o; mkdir -p $O
for cb in auto 116483 77655 58242; do
  timeout 600 python bench.py --config reddit --op gcn --col-block $cb --steps 10 --no-cpu --no-e2e > $O/gcn128_cb$cb.json 2>/dev/null
done
for cb in auto 77655 29121; do
  timeout 600 python bench.py --config reddit --op gatlayer --col-block $cb --steps 10 --no-cpu --no-e2e > $O/gatl_cb$cb.json 2>/dev/null
done
