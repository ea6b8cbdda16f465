#!/bin/bash
# same-box A/B of the GAT R-MAT / PubMed steps (libpygs.so vs libpygs_old.so)
O=gpurun_out/${1:-abg}; mkdir -p $O
timeout -s KILL 600 python -m pytest tests/test_gpu_attention.py -q 2>&1 | tail -2 > $O/pytest.txt
for i in 1 2; do
  timeout 300 python bench.py --config rmat --op gat --steps 5 --no-cpu > $O/new_$i.json 2>/dev/null
  PYG_LIBPATH=$PWD/paper_1903_02428_b200/libpygs_old.so timeout 300 python bench.py --config rmat --op gat --steps 5 --no-cpu > $O/old_$i.json 2>/dev/null
done
