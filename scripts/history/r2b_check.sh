set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r2b_gputests.log
for r in sum max; do python bench.py --config rmat --strategy atomic --reduce $r --steps 5 --warmup 3 --no-cpu --no-e2e --no-variants > gpurun_out/r2b_rmat_atomic_$r.json 2>gpurun_out/r2b_rmat_atomic_$r.err; done
python bench.py --config reddit --strategy atomic --reduce mean --steps 5 --warmup 3 --no-cpu --no-e2e --no-variants > gpurun_out/r2b_reddit_atomic_mean.json 2>gpurun_out/r2b_reddit_atomic.err
