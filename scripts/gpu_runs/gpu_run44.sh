cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 300 -x 2>&1 | tail -4
timeout 900 python scripts/sweep.py tma_sched > gpurun_out/r01_tma_sched2.jsonl 2>gpurun_out/err.log; cat gpurun_out/r01_tma_sched2.jsonl; tail -3 gpurun_out/err.log
