cd $GRAFT_REPO_ROOT
AQUA_SWEEP_BLOCK_MAJOR=1 timeout 900 python scripts/sweep.py small_chunks > gpurun_out/r01_small_chunks_bm.jsonl 2>gpurun_out/err.log; grep '"auto"' gpurun_out/r01_small_chunks_bm.jsonl | cut -c1-170; tail -2 gpurun_out/err.log
