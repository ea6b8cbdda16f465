# GAT backward: metadata read back by lane 0, unconditional slot loops
O=gpurun_out/r2o; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x 2>&1 | tail -5 > $O/attention.log
Q="--config rmat --op gat --steps 5 --no-cpu --no-e2e"
python bench.py $Q > $O/gat.json 2>$O/gat.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:"softmax|gat_|seg_|combine" --csv --log-file $O/launches_gat_rmat.csv python bench.py $Q --steps 1 --warmup 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gat_bwd_tma -c 1 -o $O/full_gat_bwd python bench.py $Q --steps 1 --warmup 1 > /dev/null 2>&1
ncu -i $O/full_gat_bwd.ncu-rep --page details --csv > $O/full_gat_bwd.details.csv 2>/dev/null
ncu -i $O/full_gat_bwd.ncu-rep --page source --csv > $O/full_gat_bwd.source.csv 2>/dev/null
ncu -i $O/full_gat_bwd.ncu-rep --page raw --csv > $O/full_gat_bwd.raw.csv 2>/dev/null
rm -f $O/full_gat_bwd.ncu-rep
