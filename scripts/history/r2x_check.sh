# MAX argmax insert by PRMT; empty rows zero-filled on a side stream concurrently with the TMA gather
O=gpurun_out/r2x; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > $O/pytest.log
for i in 1 2; do python bench.py --reduce max --steps 10 --no-cpu --no-e2e --no-variants > $O/max_$i.json 2>/dev/null; done
for red in sum max; do python bench.py --config rmat --reduce $red --steps 10 --no-cpu --no-e2e --no-variants > $O/rmat_$red.json 2>/dev/null; done
python bench.py --config rmat --op gcn --steps 10 --no-cpu --no-e2e > $O/gcn_rmat.json 2>/dev/null
python bench.py --config rmat --op gat --steps 5 --no-cpu --no-e2e > $O/gat_rmat.json 2>/dev/null
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/launches_rmat_sum.csv python bench.py --config rmat --steps 1 --warmup 2 --no-e2e --no-cpu --no-variants > /dev/null 2>&1
