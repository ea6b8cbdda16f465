#!/bin/bash
# LDG kernel vector width on narrow rows: default (V = 4 unless V = 8 fills 5% more lanes) vs forced V = 8
O=gpurun_out/r3r; mkdir -p $O
for v in 0 8; do
  for cfg in clouds pubmed; do
    PYG_SEG_VEC=$v timeout 300 python bench.py --config $cfg --steps 50 --no-e2e --no-variants --no-cpu > $O/${cfg}_v$v.json 2>/dev/null
  done
  PYG_SEG_VEC=$v timeout 600 python bench.py --config reddit --op gcn --steps 10 --no-cpu --no-e2e > $O/gcn128_v$v.json 2>/dev/null
  PYG_SEG_VEC=$v timeout 300 python bench.py --config clouds --op gat --steps 50 --no-cpu --no-e2e > $O/clouds_gat_v$v.json 2>/dev/null
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for v in 0 8; do
  PYG_SEG_VEC=$v timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/launches_clouds_v$v.csv python bench.py --config clouds --steps 1 --warmup 2 --no-cpu --no-e2e --graph off --no-variants > /dev/null 2>&1
done
