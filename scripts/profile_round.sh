#!/bin/bash
# One GPU session: parity suite, smoke, the bench lines of every config / op, ncu launch lists
# (time + DRAM bytes per launch) and one --set full capture per headline kernel, the Fig. 3 study,
# compute-sanitizer on representative tests.  Output: gpurun_out/$TAG/
set -u
TAG=${1:-r1}
O=gpurun_out/$TAG
mkdir -p $O
# gpurun copies back at most 64 MiB: every --set full report is exported to CSV (raw metrics +
# details page) and deleted; launch lists are gzipped
export_rep() {
  if [ -f "$1.ncu-rep" ]; then
    ncu -i "$1.ncu-rep" --page raw --csv > "$1.raw.csv" 2>/dev/null
    ncu -i "$1.ncu-rep" --page details --csv > "$1.details.csv" 2>/dev/null
    rm -f "$1.ncu-rep"
  fi
}
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -15 > $O/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
Q="--steps 1 --warmup 3 --no-e2e --no-cpu --no-variants"
FULL="ncu --set full --clock-control none --import-source on"
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/launches_reddit_mean.csv python bench.py $Q > /dev/null 2>&1
timeout 900 $FULL -k regex:seg_kernel -s 33 -c 1 -o $O/full_reddit_mean python bench.py $Q > /dev/null 2>&1
export_rep $O/full_reddit_mean
for red in sum max; do
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/launches_rmat_$red.csv python bench.py --config rmat --reduce $red $Q > /dev/null 2>&1
  timeout 900 $FULL -k regex:seg_tma -s 3 -c 1 -o $O/full_rmat_$red python bench.py --config rmat --reduce $red $Q > /dev/null 2>&1
  export_rep $O/full_rmat_$red
done
# atomic COO strategy: atomic throughput evidence (north_star: "atomic throughput")
timeout 900 $FULL -k regex:coo_kernel -s 3 -c 1 -o $O/full_rmat_sum_atomic python bench.py --config rmat --reduce sum --strategy atomic $Q > /dev/null 2>&1
export_rep $O/full_rmat_sum_atomic
timeout 900 $FULL -k regex:coo_tile -s 19 -c 1 -o $O/full_reddit_mean_atomic python bench.py --strategy atomic $Q > /dev/null 2>&1
export_rep $O/full_reddit_mean_atomic
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/launches_reddit_mean_atomic.csv python bench.py --strategy atomic $Q > /dev/null 2>&1
for red in sum max; do
  timeout 600 python bench.py --config rmat --reduce $red --steps 10 --no-e2e --no-cpu --no-variants > $O/bench_rmat_$red.json 2> $O/bench_rmat_$red.err
  timeout 600 python bench.py --config rmat --reduce $red --strategy atomic --steps 5 --no-e2e --no-cpu --no-variants > $O/bench_rmat_${red}_atomic.json 2> $O/bench_rmat_${red}_atomic.err
done
timeout 600 python bench.py --strategy atomic --steps 5 --no-cpu --no-variants > $O/bench_reddit_mean_atomic.json 2> $O/bench_reddit_mean_atomic.err
timeout 600 python bench.py --strategy atomic --reduce max --steps 5 --no-e2e --no-cpu --no-variants > $O/bench_reddit_max_atomic.json 2> $O/bench_reddit_max_atomic.err
for cfg in pubmed clouds cora; do
  timeout 300 python bench.py --config $cfg --strategy atomic --steps 50 --no-e2e --no-variants --no-cpu > $O/bench_${cfg}_atomic.json 2> $O/bench_${cfg}_atomic.err
done
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/l2red scripts/l2red.cu && timeout 300 /tmp/l2red > $O/l2red.json 2> $O/l2red.err
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/l2peak scripts/l2peak.cu && timeout 300 /tmp/l2peak > $O/l2peak.json 2> $O/l2peak.err
for cfg in pubmed clouds cora; do  # pubmed = GCN fwd+bwd
  timeout 300 python bench.py --config $cfg --steps 50 --no-e2e --no-variants > $O/bench_$cfg.json 2> $O/bench_$cfg.err
done
# NEXT rows: GAT (NEXT-1), APPNP and the GCN layer with the tcgen05 transform (NEXT-2)
for cfg in rmat pubmed; do
  timeout 600 python bench.py --config $cfg --op gat --steps 10 > $O/bench_gat_$cfg.json 2> $O/bench_gat_$cfg.err
done
for cfg in reddit pubmed; do
  timeout 600 python bench.py --config $cfg --op appnp --steps 5 > $O/bench_appnp_$cfg.json 2> $O/bench_appnp_$cfg.err
done
for cfg in reddit rmat pubmed; do
  timeout 600 python bench.py --config $cfg --op gcn --steps 10 > $O/bench_gcn_$cfg.json 2> $O/bench_gcn_$cfg.err
done
timeout 600 python bench.py --op gcn --hidden 512 --steps 10 > $O/bench_gcn512.json 2> $O/bench_gcn512.err
for cfg in rmat reddit pubmed; do
  timeout 600 python bench.py --config $cfg --op gatlayer --steps 10 > $O/bench_gatlayer_$cfg.json 2> $O/bench_gatlayer_$cfg.err
done
timeout 600 python bench.py --reduce max --steps 10 --no-e2e --no-cpu --no-variants > $O/bench_reddit_max.json 2> $O/bench_reddit_max.err
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/launches_reddit_max.csv python bench.py --reduce max $Q > /dev/null 2>&1
timeout 900 $FULL -k regex:seg_kernel -s 12 -c 1 -o $O/full_reddit_max python bench.py --reduce max $Q > /dev/null 2>&1
export_rep $O/full_reddit_max
timeout 900 $FULL -k regex:"gat_(bwd|fwd)_tma" -c 2 -o $O/full_gat_rmat python bench.py --config rmat --op gat $Q > /dev/null 2>&1
export_rep $O/full_gat_rmat
timeout 600 ncu --metrics $M --clock-control none -k regex:"softmax|seg_|combine|gat_" --csv --log-file $O/launches_gat_rmat.csv python bench.py --config rmat --op gat $Q > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:"tf32|seg_|combine|deg_rsqrt" --csv --log-file $O/launches_gcn_reddit.csv python bench.py --config reddit --op gcn $Q > /dev/null 2>&1
timeout 900 $FULL -k regex:tf32 -s 1 -c 1 -o $O/full_tf32_reddit python bench.py --config reddit --op gcn $Q > /dev/null 2>&1
export_rep $O/full_tf32_reddit
timeout 600 python scripts/fig3.py --out $O/fig3.json > $O/fig3.log 2>&1
# (compute-sanitizer is closed on this pool since round 2's last session: runs under it left GPUs
# needing a reset.  The round-2 memcheck / racecheck logs are profiles/r2a_sanitizer_* and
# r2ab_sanitizer_*; memory safety of later kernels rests on bounds-checked parity tests.)
gzip -f $O/launches_*.csv
