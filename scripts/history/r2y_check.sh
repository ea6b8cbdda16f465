# GAT: forward aggregation loop not unrolled (one flush path), reciprocal per chunk; occupancy sweep
O=gpurun_out/r2y; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_attention.py -q -x 2>&1 | tail -3 > $O/attention.log
Q="--config rmat --op gat --steps 5 --no-cpu --no-e2e"
python bench.py $Q > $O/gat.json 2>$O/gat.err
PYG_GAT_SM_KB=227 python bench.py $Q > $O/gat_bsm227.json 2>/dev/null
PYG_GAT_WARPS=4 PYG_GAT_SM_KB=200 python bench.py $Q > $O/gat_w4_bsm200.json 2>/dev/null
PYG_GAT_FWD_SM_KB=200 python bench.py $Q > $O/gat_fsm200.json 2>/dev/null
PYG_GAT_FWD_SM_KB=120 python bench.py $Q > $O/gat_fsm120.json 2>/dev/null
PYG_GAT_FWD_WARP_KB=8 python bench.py $Q > $O/gat_fwk8.json 2>/dev/null
PYG_GAT_WARP_KB=14 PYG_GAT_SM_KB=227 python bench.py $Q > $O/gat_bwk14.json 2>/dev/null
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:"gat_|seg_|combine" --csv --log-file $O/launches_gat_rmat.csv python bench.py $Q --steps 1 --warmup 2 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_halo_push.py tests/test_gpu_bench_multi.py tests/test_gpu_dist.py -q -x 2>&1 | tail -3 > $O/multi.log
python bench.py --config reddit --op gatlayer --steps 10 --no-cpu --no-e2e > $O/gatlayer_reddit_blocked.json 2>$O/gatlayer_reddit_blocked.err
python bench.py --config reddit --op gatlayer --col-block 0 --steps 10 --no-cpu --no-e2e > $O/gatlayer_reddit_unblocked.json 2>/dev/null
python bench.py --config rmat --op gatlayer --steps 10 --no-cpu --no-e2e > $O/gatlayer_rmat.json 2>/dev/null
