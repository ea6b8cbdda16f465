# blocked GAT forward with grouped weights; empty-row fill with coalesced args; clouds / PubMed GAT regressions
O=gpurun_out/r2z; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3 > $O/tests.log
python bench.py --config reddit --op gatlayer --steps 10 --no-cpu --no-e2e > $O/gatlayer_reddit.json 2>$O/gatlayer_reddit.err
python bench.py --config rmat --op gat --steps 5 --no-cpu --no-e2e > $O/gat_rmat.json 2>/dev/null
python bench.py --config pubmed --op gat --steps 50 --no-cpu --no-e2e > $O/gat_pubmed.json 2>/dev/null
python bench.py --config rmat --reduce max --steps 10 --no-cpu --no-e2e --no-variants > $O/rmat_max.json 2>/dev/null
python bench.py --config clouds --steps 50 --no-cpu --no-e2e > $O/clouds.json 2>/dev/null
python bench.py --config cora --steps 50 --no-cpu --no-e2e > $O/cora.json 2>/dev/null
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/launches_clouds.csv python bench.py --config clouds --steps 1 --warmup 2 --no-cpu --no-e2e --graph off > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:"gat_" --csv --log-file $O/launches_gatlayer_reddit.csv python bench.py --config reddit --op gatlayer --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
timeout 300 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_attention.py -q -x -k "far_logits and 1" > $O/racecheck_far.log 2>&1
timeout 300 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_attention.py -q -x -k "far_logits or source_blocked" > $O/memcheck_far.log 2>&1
