#!/bin/bash
# ncu --set full of coo_tile_kernel (Reddit mean), default bench line (e2e D2H overlap), Reddit max
# source-block size sweep, atomic tests
O=gpurun_out/r3g; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "atomic or coo or scatter_random" 2>&1 | tail -3 > $O/tests.txt
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
Q="--steps 5 --no-e2e --no-cpu --no-variants"
timeout 600 python bench.py --strategy atomic --reduce max $Q > $O/reddit_max_atomic.json 2>/dev/null
for cb in 15000 18000 26000 32000; do
  timeout 600 python bench.py --reduce max --col-block $cb --steps 10 --no-e2e --no-cpu --no-variants > $O/reddit_max_cb$cb.json 2>/dev/null
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:coo_tile -s 1 -c 1 -o $O/full_tile python bench.py --strategy atomic --steps 1 --warmup 1 --no-e2e --no-cpu --no-variants > /dev/null 2>&1
ncu -i $O/full_tile.ncu-rep --page raw --csv > $O/full_tile.raw.csv 2>/dev/null
ncu -i $O/full_tile.ncu-rep --page details --csv > $O/full_tile.details.csv 2>/dev/null
ncu -i $O/full_tile.ncu-rep --page source --csv > $O/full_tile.source.csv 2>/dev/null
rm -f $O/*.ncu-rep
