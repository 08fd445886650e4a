cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r02_gpu_suite7.log 2>&1; echo "suite rc $?"; tail -3 gpurun_out/r02_gpu_suite7.log
AQUA_SWEEP_S=512,1024,2048 AQUA_SWEEP_ENGINES=auto timeout 900 python scripts/sweep.py small_chunks2 > gpurun_out/r02_small_chunks_auto4.jsonl 2>gpurun_out/err.log; cut -c1-250 gpurun_out/r02_small_chunks_auto4.jsonl; tail -2 gpurun_out/err.log
