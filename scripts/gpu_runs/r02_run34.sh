cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r02_gpu_suite8.log 2>&1; echo "suite rc $?"; tail -3 gpurun_out/r02_gpu_suite8.log
timeout 600 python scripts/sweep.py latency > gpurun_out/r02_latency.jsonl 2>gpurun_out/err.log; cat gpurun_out/r02_latency.jsonl; tail -2 gpurun_out/err.log
