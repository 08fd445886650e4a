cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r02_gpu_suite4.log 2>&1; echo "suite rc $?"; tail -3 gpurun_out/r02_gpu_suite4.log
AQUA_SWEEP_S=512,1024,2048,4096,8192,32768 timeout 900 python scripts/sweep.py small_chunks2 > gpurun_out/r02_small_chunks_final2.jsonl 2>gpurun_out/err.log; grep auto gpurun_out/r02_small_chunks_final2.jsonl | cut -c1-220; tail -2 gpurun_out/err.log
