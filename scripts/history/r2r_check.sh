# GAT backward v2b: rotated conflict-free head chunks, NB template, sequential chunk sums
O=gpurun_out/r2r; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x 2>&1 | tail -25 > $O/attention.log
Q="--config rmat --op gat --steps 5 --no-cpu --no-e2e"
python bench.py $Q > $O/gat.json 2>$O/gat.err
PYG_GAT_FUSED=0 python bench.py $Q > $O/gat_unfused.json 2>/dev/null
python bench.py --config rmat --op gatlayer --steps 5 --no-cpu --no-e2e > $O/gatlayer_rmat.json 2>/dev/null
python bench.py --config reddit --op gatlayer --steps 5 --no-cpu --no-e2e > $O/gatlayer_reddit.json 2>/dev/null
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:"softmax|gat_|seg_|combine" --csv --log-file $O/launches_gat_rmat.csv python bench.py $Q --steps 1 --warmup 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gat_(bwd|fwd)_tma" -c 2 -o $O/full_gat python bench.py $Q --steps 1 --warmup 1 > /dev/null 2>&1
ncu -i $O/full_gat.ncu-rep --page details --csv > $O/full_gat.details.csv 2>/dev/null
ncu -i $O/full_gat.ncu-rep --page raw --csv > $O/full_gat.raw.csv 2>/dev/null
rm -f $O/full_gat.ncu-rep
