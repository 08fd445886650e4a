cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_mixed_fuzz.py -q -m gpu -x > gpurun_out/r02_mixed_fuzz.log 2>&1; echo "rc $?"; tail -3 gpurun_out/r02_mixed_fuzz.log
AQUA_FUZZ_SEEDS=60 AQUA_FUZZ_OPS=80 timeout 2400 python -m pytest tests/test_gpu_mixed_fuzz.py -q -m gpu -x > gpurun_out/r02_mixed_fuzz_long.log 2>&1; echo "rc $?"; tail -30 gpurun_out/r02_mixed_fuzz_long.log
