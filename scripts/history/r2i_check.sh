# the row-staged bulk-copy kernel: parity vs LDG + oracle, then Reddit timings (bulk auto = MAX)
O=gpurun_out/r2i; mkdir -p $O
python -m pytest tests/test_gpu_parity.py -q -x -k "bulk or blocked" 2>&1 | tail -15 > $O/tests.log
python -m pytest tests/test_gpu_configs.py -q -x -k "blocked" 2>&1 | tail -5 >> $O/tests.log
python bench.py --reduce max --steps 10 --no-cpu --no-e2e --no-variants > $O/reddit_max_bulk.json 2>$O/reddit_max_bulk.err
PYG_SEG_BULK=0 python bench.py --reduce max --steps 10 --no-cpu --no-e2e --no-variants > $O/reddit_max_ldg.json 2>/dev/null
PYG_SEG_BULK=1 python bench.py --reduce mean --steps 10 --no-cpu --no-e2e --no-variants > $O/reddit_mean_bulk.json 2>/dev/null
python bench.py --reduce mean --steps 10 --no-cpu --no-e2e --no-variants > $O/reddit_mean_ldg.json 2>/dev/null
PYG_SEG_BULK=1 python bench.py --op gcn --hidden 512 --steps 10 --no-cpu --no-e2e > $O/gcn512_bulk.json 2>/dev/null
python bench.py --op gcn --hidden 512 --steps 10 --no-cpu --no-e2e > $O/gcn512_ldg.json 2>/dev/null
for kb in 6 12 16; do PYG_BULK_WARP_KB=$kb python bench.py --reduce max --steps 10 --no-cpu --no-e2e --no-variants > $O/reddit_max_bulk_kb$kb.json 2>/dev/null; done
python bench.py --config pubmed --steps 20 --no-cpu --no-e2e > $O/pubmed.json 2>/dev/null
