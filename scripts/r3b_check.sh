#!/bin/bash
# atomic COO with L2 column tiles: parity (child process, 1 MB budget) + Reddit / R-MAT atomic lines
O=gpurun_out/r3b; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_coo_tiles.py tests/test_gpu_configs.py tests/test_gpu_parity.py -q -x -k "coo_tiles or atomic or scatter_random or propagate_random or backward" 2>&1 | tail -15 > $O/tests.txt
Q="--steps 5 --no-e2e --no-cpu --no-variants"
for red in mean sum max; do
  for mb in 72 48 100; do
    PYG_COO_L2_MB=$mb timeout 600 python bench.py --strategy atomic --reduce $red $Q > $O/reddit_${red}_atomic_$mb.json 2> $O/reddit_${red}_atomic_$mb.err
  done
done
timeout 600 python bench.py --config rmat --reduce sum --strategy atomic $Q > $O/rmat_sum_atomic.json 2> $O/rmat_sum_atomic.err
timeout 300 python bench.py --config pubmed --strategy atomic --steps 50 --no-e2e --no-variants > $O/pubmed_atomic.json 2> $O/pubmed_atomic.err
PYG_COO_L2_MB=0 timeout 300 python bench.py --config pubmed --strategy atomic --steps 50 --no-e2e --no-variants > $O/pubmed_atomic_notile.json 2> $O/pubmed_atomic_notile.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
timeout 600 ncu --metrics $M --clock-control none -k regex:coo_kernel --csv --log-file $O/launches_reddit_mean_atomic.csv python bench.py --strategy atomic --steps 1 --warmup 1 --no-e2e --no-cpu --no-variants > /dev/null 2>&1
