cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 300 -x 2>&1 | tail -3
timeout 900 python scripts/sweep.py small_chunks > gpurun_out/r01_small_chunks2.jsonl 2>gpurun_out/err.log; grep auto gpurun_out/r01_small_chunks2.jsonl
timeout 900 python scripts/sweep.py hybrid > gpurun_out/r01_hybrid3.jsonl 2>>gpurun_out/err.log; grep auto gpurun_out/r01_hybrid3.jsonl; tail -3 gpurun_out/err.log
