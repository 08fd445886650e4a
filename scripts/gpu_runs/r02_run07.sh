cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "staged or pack" > gpurun_out/r02_staged_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/r02_staged_tests.log
timeout 900 python scripts/sweep.py small_chunks2 > gpurun_out/r02_small_chunks3.jsonl 2>gpurun_out/err.log; tail -2 gpurun_out/err.log
