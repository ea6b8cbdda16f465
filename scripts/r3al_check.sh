#!/bin/bash
O=gpurun_out/r3al; mkdir -p $O
for i in 1 2; do
  timeout 600 python bench.py --config reddit --op gatlayer --steps 10 --no-e2e --no-cpu > $O/gatl_auto_$i.json 2>/dev/null
  timeout 600 python bench.py --config reddit --op gatlayer --col-block 46593 --steps 10 --no-e2e --no-cpu > $O/gatl_5p_$i.json 2>/dev/null
done
timeout 600 python bench.py --config pubmed --op gatlayer --steps 20 --no-e2e --no-cpu > $O/gatl_pubmed.json 2>/dev/null
timeout 600 python bench.py --config rmat --op gatlayer --steps 5 --no-e2e --no-cpu > $O/gatl_rmat.json 2>/dev/null
