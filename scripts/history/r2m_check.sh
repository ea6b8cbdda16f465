# one-pass GAT backward: parity, ring / smem sweep, ncu full; bulk kernel (coalesced index windows) parity + Reddit max A/B
O=gpurun_out/r2m; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x 2>&1 | tail -5 > $O/attention.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -40 > $O/parity.log
Q="--config rmat --op gat --steps 5 --no-cpu --no-e2e"
python bench.py $Q > $O/gat_w10_s160.json 2>$O/gat.err
PYG_GAT_SM_KB=200 python bench.py $Q > $O/gat_w10_s200.json 2>/dev/null
PYG_GAT_WARP_KB=14 PYG_GAT_SM_KB=227 python bench.py $Q > $O/gat_w14_s227.json 2>/dev/null
PYG_GAT_WARP_KB=19 PYG_GAT_SM_KB=160 python bench.py $Q > $O/gat_w19_s160.json 2>/dev/null
python bench.py --reduce max --steps 10 --no-cpu --no-e2e --no-variants > $O/reddit_max_ldg.json 2>/dev/null
PYG_SEG_BULK=1 python bench.py --reduce max --steps 10 --no-cpu --no-e2e --no-variants > $O/reddit_max_bulk.json 2>/dev/null
PYG_SEG_BULK=1 PYG_BULK_WARP_KB=16 python bench.py --reduce max --steps 10 --no-cpu --no-e2e --no-variants > $O/reddit_max_bulk16.json 2>/dev/null
PYG_SEG_BULK=1 python bench.py --reduce mean --steps 10 --no-cpu --no-e2e --no-variants > $O/reddit_mean_bulk.json 2>/dev/null
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:"softmax|gat_|seg_|combine" --csv --log-file $O/launches_gat_rmat.csv python bench.py $Q --steps 1 --warmup 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gat_bwd_tma -c 1 -o $O/full_gat_bwd python bench.py $Q --steps 1 --warmup 1 > /dev/null 2>&1
ncu -i $O/full_gat_bwd.ncu-rep --page raw --csv > $O/full_gat_bwd.raw.csv 2>/dev/null
ncu -i $O/full_gat_bwd.ncu-rep --page details --csv > $O/full_gat_bwd.details.csv 2>/dev/null
ncu -i $O/full_gat_bwd.ncu-rep --page source --csv > $O/full_gat_bwd.source.csv 2>/dev/null
rm -f $O/full_gat_bwd.ncu-rep
