cd $GRAFT_REPO_ROOT
AQUA_SWEEP_S=512,1024,2048,4096,8192,32768 AQUA_SWEEP_ENGINES=auto timeout 900 python scripts/sweep.py small_chunks2 > gpurun_out/r02_small_chunks_auto3.jsonl 2>gpurun_out/err.log; cut -c1-250 gpurun_out/r02_small_chunks_auto3.jsonl; tail -2 gpurun_out/err.log
AQUA_SWEEP_BLOCK_MAJOR=1 timeout 900 python scripts/sweep.py small_chunks > gpurun_out/r02_small_chunks_bm.jsonl 2>>gpurun_out/err.log; grep '"auto"' gpurun_out/r02_small_chunks_bm.jsonl | cut -c1-200
