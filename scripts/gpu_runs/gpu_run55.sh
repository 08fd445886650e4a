cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 300 -x 2>&1 | tail -4
timeout 900 python scripts/sweep.py hybrid > gpurun_out/r01_hybrid.jsonl 2>gpurun_out/err.log; cat gpurun_out/r01_hybrid.jsonl; tail -3 gpurun_out/err.log
