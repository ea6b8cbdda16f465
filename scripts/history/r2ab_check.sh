# bad-row lists deduplicated by a warp ballot; full GPU suite; memcheck of the GAT TMA / blocked kernels
O=gpurun_out/r2ab; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > $O/pytest.log
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 99 python -m pytest tests/test_gpu_attention.py -q -x -k "far_logits or source_blocked or one_pass or (backward and rmat_h4c16) or (factored and rmat_h4c16)" > $O/memcheck_gat.log 2>&1; echo "exit=$?" >> $O/memcheck_gat.log
timeout 600 compute-sanitizer --tool racecheck --error-exitcode 99 python -m pytest tests/test_gpu_attention.py -q -x -k "source_blocked or one_pass or (backward and rmat_h4c16 and factored)" > $O/racecheck_gat.log 2>&1; echo "exit=$?" >> $O/racecheck_gat.log
python bench.py --config rmat --op gat --steps 5 --no-cpu --no-e2e > $O/gat_rmat.json 2>/dev/null
python bench.py --config reddit --op gatlayer --steps 10 --no-cpu --no-e2e > $O/gatlayer_reddit.json 2>/dev/null
python bench.py --config pubmed --op gat --steps 50 --no-cpu --no-e2e > $O/gat_pubmed.json 2>/dev/null
