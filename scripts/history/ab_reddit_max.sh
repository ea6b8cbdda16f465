#!/bin/bash
# same-box A/B of the Reddit max variant (libpygs.so vs libpygs_old.so)
O=gpurun_out/${1:-abm}; mkdir -p $O
timeout -s KILL 900 python -m pytest tests -m gpu -q -k "max or propagate or scatter or source_blocked" 2>&1 | tail -2 > $O/pytest.txt
for i in 1 2; do
  timeout 300 python bench.py --reduce max --steps 10 --no-e2e --no-cpu --no-variants > $O/new_$i.json 2>/dev/null
  PYG_LIBPATH=$PWD/paper_1903_02428_b200/libpygs_old.so timeout 300 python bench.py --reduce max --steps 10 --no-e2e --no-cpu --no-variants > $O/old_$i.json 2>/dev/null
done
timeout 300 python bench.py --config clouds --steps 50 --no-e2e --no-variants > $O/clouds.json 2>/dev/null
PYG_LIBPATH=$PWD/paper_1903_02428_b200/libpygs_old.so timeout 300 python bench.py --config clouds --steps 50 --no-e2e --no-variants > $O/clouds_old.json 2>/dev/null
