#!/bin/bash
O=gpurun_out/r3am; mkdir -p $O
for cb in 21179 15000 29121; do
  timeout 900 python bench.py --config reddit --op appnp --col-block $cb --steps 3 --no-e2e --no-cpu > $O/appnp_cb$cb.json 2>/dev/null
done
