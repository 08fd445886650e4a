cd $GRAFT_REPO_ROOT
AQUA_SWEEP_S=512,1024,2048,4096 AQUA_SWEEP_ENGINES=auto,ring AQUA_SWEEP_RING_STAGES=0,4,6,8,12 timeout 900 python scripts/sweep.py small_chunks2 > gpurun_out/r02_small_stages.jsonl 2>gpurun_out/err.log; tail -2 gpurun_out/err.log
