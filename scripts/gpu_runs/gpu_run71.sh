cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 300 -x 2>&1 | tail -3
timeout 900 python scripts/sweep.py small_chunks > gpurun_out/r01_small_chunks4.jsonl 2>gpurun_out/err.log; grep -v '"sched": 16' gpurun_out/r01_small_chunks4.jsonl | cut -c1-160; tail -2 gpurun_out/err.log
