cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 300 -x 2>&1 | tail -3
timeout 900 python scripts/sweep.py small_chunks > gpurun_out/r01_small_chunks3.jsonl 2>gpurun_out/err.log; cat gpurun_out/r01_small_chunks3.jsonl | cut -c1-160; tail -2 gpurun_out/err.log
