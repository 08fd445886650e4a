cd $GRAFT_REPO_ROOT
timeout 600 python scripts/sweep.py exchange > gpurun_out/r01_exchange2.jsonl 2>gpurun_out/err.log; cat gpurun_out/r01_exchange2.jsonl; tail -2 gpurun_out/err.log
