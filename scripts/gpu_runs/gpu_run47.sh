cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 300 -x 2>&1 | tail -4
AQUA_SWEEP_SCHED="0:0,1:0,2:0,4:0,8:0,16:0,-1:0,-2:0,-4:0" timeout 1200 python scripts/sweep.py tma_sched > gpurun_out/r01_tma_sched5.jsonl 2>gpurun_out/err.log; cat gpurun_out/r01_tma_sched5.jsonl | cut -c1-150; tail -3 gpurun_out/err.log
