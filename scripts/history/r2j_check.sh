# re-entry check of the round-2 state: GPU suite, smoke, headline + variant bench lines, launch list
O=gpurun_out/r2j; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -25 > $O/pytest.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/reddit_mean.json 2>$O/reddit_mean.err
python bench.py --reduce max --steps 10 --no-cpu --no-e2e --no-variants > $O/reddit_max.json 2>/dev/null
python bench.py --config rmat --reduce sum --steps 10 --no-e2e --no-variants > $O/rmat_sum.json 2>/dev/null
python bench.py --config rmat --strategy atomic --reduce sum --steps 5 --no-cpu --no-e2e --no-variants > $O/rmat_atomic_sum.json 2>/dev/null
python bench.py --config rmat --strategy atomic --reduce max --steps 5 --no-cpu --no-e2e --no-variants > $O/rmat_atomic_max.json 2>/dev/null
python bench.py --strategy atomic --steps 5 --no-cpu --no-e2e --no-variants > $O/reddit_atomic_mean.json 2>/dev/null
python bench.py --op gcn --hidden 512 --steps 10 --no-cpu --no-e2e > $O/reddit_gcn512.json 2>/dev/null
python bench.py --config rmat --op gat --steps 5 --no-cpu --no-e2e > $O/gat_rmat.json 2>/dev/null
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/launches_reddit_mean.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-variants > /dev/null 2>&1
