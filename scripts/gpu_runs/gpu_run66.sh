cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 300 -x 2>&1 | tail -3
timeout 600 python scripts/sweep.py latency > gpurun_out/r01_latency_small.jsonl 2>gpurun_out/err.log; cat gpurun_out/r01_latency_small.jsonl | cut -c1-250
