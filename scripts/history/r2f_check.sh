O=gpurun_out/r2f; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > $O/pytest.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1
python bench.py --steps 10 > $O/reddit_mean.json 2>$O/reddit_mean.err
python bench.py --reduce max --steps 10 --no-cpu --no-e2e --no-variants > $O/reddit_max.json 2>/dev/null
python bench.py --config rmat --strategy atomic --reduce sum --steps 5 --no-cpu --no-e2e --no-variants > $O/rmat_atomic_sum.json 2>/dev/null
python bench.py --config rmat --strategy atomic --reduce max --steps 5 --no-cpu --no-e2e --no-variants > $O/rmat_atomic_max.json 2>/dev/null
python bench.py --op gcn --hidden 512 --steps 10 --no-cpu --no-e2e > $O/reddit_gcn512.json 2>$O/reddit_gcn512.err
python bench.py --op gcn --hidden 128 --steps 10 --no-cpu --no-e2e > $O/reddit_gcn128.json 2>/dev/null
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/l2peak scripts/l2peak.cu && /tmp/l2peak > $O/l2peak.json 2>&1
