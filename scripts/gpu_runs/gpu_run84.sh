cd $GRAFT_REPO_ROOT
timeout 600 python scripts/sweep.py rate > gpurun_out/r01_rate.jsonl 2>gpurun_out/err.log; cat gpurun_out/r01_rate.jsonl; tail -2 gpurun_out/err.log
