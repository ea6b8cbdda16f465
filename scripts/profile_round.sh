#!/bin/bash
# One GPU session: parity suite, smoke, default bench, ncu launch lists (time + DRAM bytes per
# launch) and one --set full capture per headline kernel.  Output: gpurun_out/$TAG/
set -u
TAG=${1:-r1}
O=gpurun_out/$TAG
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -15 > $O/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
Q="--steps 1 --warmup 3 --no-e2e --no-cpu --no-variants"
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/launches_reddit_mean.csv python bench.py $Q > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_kernel -s 33 -c 1 -o $O/full_reddit_mean python bench.py $Q > /dev/null 2>&1
for red in sum max; do
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/launches_rmat_$red.csv python bench.py --config rmat --reduce $red $Q > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_tma -s 3 -c 1 -o $O/full_rmat_sum python bench.py --config rmat --reduce sum $Q > /dev/null 2>&1
for red in sum max; do
  timeout 600 python bench.py --config rmat --reduce $red --steps 10 --no-e2e --no-cpu --no-variants > $O/bench_rmat_$red.json 2> $O/bench_rmat_$red.err
  timeout 600 python bench.py --config rmat --reduce $red --strategy atomic --steps 5 --no-e2e --no-cpu --no-variants > $O/bench_rmat_${red}_atomic.json 2> $O/bench_rmat_${red}_atomic.err
done
for cfg in pubmed clouds cora; do  # pubmed = GCN fwd+bwd
  timeout 300 python bench.py --config $cfg --steps 50 --no-e2e --no-variants > $O/bench_$cfg.json 2> $O/bench_$cfg.err
done
# memory-safety evidence: compute-sanitizer memcheck / racecheck on representative small tests
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -q -x \
  -k "scatter_printed or split_hub or (tma_pipeline and 128) or (source_blocked and 37) or collate or concat_and_edge_attr or backward" \
  > $O/sanitizer_memcheck.txt 2>&1; echo "exit=$?" >> $O/sanitizer_memcheck.txt
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -q -x \
  -k "(tma_pipeline and 128) or split_hub" > $O/sanitizer_racecheck.txt 2>&1; echo "exit=$?" >> $O/sanitizer_racecheck.txt
