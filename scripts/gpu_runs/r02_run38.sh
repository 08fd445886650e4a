cd $GRAFT_REPO_ROOT
timeout 600 python scripts/sweep.py small_calls > gpurun_out/r02_small_calls.jsonl 2>gpurun_out/err.log; cat gpurun_out/r02_small_calls.jsonl; tail -3 gpurun_out/err.log
