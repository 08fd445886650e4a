cd $GRAFT_REPO_ROOT
timeout 900 python scripts/sweep.py small_chunks > gpurun_out/r01_small_chunks.jsonl 2>gpurun_out/err.log; cat gpurun_out/r01_small_chunks.jsonl; tail -3 gpurun_out/err.log
