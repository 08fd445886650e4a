cd $GRAFT_REPO_ROOT
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 2400 $CS --tool memcheck --leak-check full python -m pytest tests/test_gpu_mixed_fuzz.py -q -m gpu -p no:cacheprovider > gpurun_out/r02_sanitizer_memcheck_mixed.log 2>&1; echo "memcheck rc $?"; grep -E "ERROR SUMMARY|LEAK SUMMARY|passed|failed" gpurun_out/r02_sanitizer_memcheck_mixed.log | tail -4
timeout 2400 $CS --tool racecheck python -m pytest tests/test_gpu_mixed_fuzz.py -q -m gpu -p no:cacheprovider -k "seed0 or seed1" > gpurun_out/r02_sanitizer_racecheck_mixed.log 2>&1; echo "racecheck rc $?"; grep -E "RACECHECK SUMMARY|ERROR SUMMARY|passed|failed" gpurun_out/r02_sanitizer_racecheck_mixed.log | tail -4
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r02_gpu_suite9.log 2>&1; echo "suite rc $?"; tail -2 gpurun_out/r02_gpu_suite9.log
