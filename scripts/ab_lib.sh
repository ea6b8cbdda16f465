#!/bin/bash
# A/B of two builds of the library on the same box: libpygs.so (new) vs libpygs_old.so (PYG_LIBPATH)
O=gpurun_out/${1:-ab}
mkdir -p $O
timeout -s KILL 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/pytest.txt
for i in 1 2; do
  for red in sum max; do
    timeout 300 python bench.py --config rmat --reduce $red --steps 10 --no-e2e --no-cpu --no-variants > $O/new_${red}_$i.json 2>/dev/null
    PYG_LIBPATH=$PWD/paper_1903_02428_b200/libpygs_old.so timeout 300 python bench.py --config rmat --reduce $red --steps 10 --no-e2e --no-cpu --no-variants > $O/old_${red}_$i.json 2>/dev/null
  done
done
timeout 400 python bench.py --steps 10 --no-variants > $O/reddit_default.json 2>/dev/null
