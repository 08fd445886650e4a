cd $GRAFT_REPO_ROOT
AQUA_SWEEP_SCHED="0:0,1:0,2:0,3:0,4:0,6:0" AQUA_SWEEP_CTAS=0 AQUA_SWEEP_STAGES="0,4,5" timeout 1200 python scripts/sweep.py tma_sched > gpurun_out/r01_tma_sched6.jsonl 2>gpurun_out/err.log; cat gpurun_out/r01_tma_sched6.jsonl | cut -c1-190; tail -3 gpurun_out/err.log
