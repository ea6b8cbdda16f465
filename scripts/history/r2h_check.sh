# A/B: GAT softmax positions per thread (PU 4 default / 2 / 1); F=512 aggregation V=8 vs V=4; Reddit max
O=gpurun_out/r2h; mkdir -p $O
L=$PWD/paper_1903_02428_b200
python bench.py --reduce max --steps 10 --no-cpu --no-e2e --no-variants > $O/reddit_max.json 2>/dev/null
python bench.py --op gcn --hidden 512 --steps 10 --no-cpu --no-e2e > $O/gcn512_v8.json 2>/dev/null
PYG_SEG_VEC=4 python bench.py --op gcn --hidden 512 --steps 10 --no-cpu --no-e2e > $O/gcn512_v4.json 2>/dev/null
for i in 1 2; do
python bench.py --config rmat --op gat --steps 5 --no-cpu --no-e2e > $O/gat_pu4_$i.json 2>/dev/null
PYG_LIBPATH=$L/libpygs_pu2.so python bench.py --config rmat --op gat --steps 5 --no-cpu --no-e2e > $O/gat_pu2_$i.json 2>/dev/null
PYG_LIBPATH=$L/libpygs_pu1.so python bench.py --config rmat --op gat --steps 5 --no-cpu --no-e2e > $O/gat_pu1_$i.json 2>/dev/null
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -k regex:"softmax|gat_|seg_|combine" --csv --log-file $O/launches_gat_rmat.csv python bench.py --config rmat --op gat --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
python -m pytest tests/test_gpu_attention.py -q 2>&1 | tail -2 > $O/tests_attention.log
