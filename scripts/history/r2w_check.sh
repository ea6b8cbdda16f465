# packed-argmax MAX (unweighted instantiation without the multiply) + GPU suite; ncu of a Reddit max pass;
# GAT fwd / bwd per-CUDA-line ncu source view
O=gpurun_out/r2w; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -8 > $O/pytest.log
for i in 1 2; do python bench.py --reduce max --steps 10 --no-cpu --no-e2e --no-variants > $O/max_$i.json 2>/dev/null; done
python bench.py --config rmat --reduce max --steps 10 --no-cpu --no-e2e --no-variants > $O/rmat_max.json 2>/dev/null
FULL="ncu --set full --clock-control none --import-source on"
Q="--steps 1 --warmup 1 --no-e2e --no-cpu --no-variants"
timeout 900 $FULL -k regex:seg_kernel -s 12 -c 1 -o $O/full_reddit_max python bench.py --reduce max $Q > /dev/null 2>&1
for r in full_reddit_max; do
  ncu -i $O/$r.ncu-rep --page details --csv > $O/$r.details.csv 2>/dev/null
  ncu -i $O/$r.ncu-rep --page raw --csv > $O/$r.raw.csv 2>/dev/null
  ncu -i $O/$r.ncu-rep --page source --print-source cuda --csv > $O/$r.cuda.csv 2>/dev/null
  rm -f $O/$r.ncu-rep
done
G="--config rmat --op gat --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 900 $FULL -k regex:"gat_(bwd|fwd)_tma" -c 2 -o $O/full_gat python bench.py $G > /dev/null 2>&1
ncu -i $O/full_gat.ncu-rep --page source --print-source cuda --csv > $O/full_gat.cuda.csv 2>/dev/null
ncu -i $O/full_gat.ncu-rep --page raw --csv > $O/full_gat.raw.csv 2>/dev/null
rm -f $O/full_gat.ncu-rep
