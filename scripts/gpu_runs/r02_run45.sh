cd $GRAFT_REPO_ROOT
CS=/usr/local/cuda/bin/compute-sanitizer
AQUA_FUZZ_SEEDS=2 timeout 2400 $CS --tool racecheck python -m pytest tests/test_gpu_mixed_fuzz.py -q -m gpu -p no:cacheprovider > gpurun_out/r02_sanitizer_racecheck_mixed.log 2>&1; echo "racecheck rc $?"; grep -E "RACECHECK SUMMARY|ERROR SUMMARY|passed|failed" gpurun_out/r02_sanitizer_racecheck_mixed.log | tail -4
AQUA_FUZZ_SEEDS=1 timeout 2400 $CS --tool synccheck python -m pytest tests/test_gpu_mixed_fuzz.py -q -m gpu -p no:cacheprovider > gpurun_out/r02_sanitizer_synccheck_mixed.log 2>&1; echo "synccheck rc $?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/r02_sanitizer_synccheck_mixed.log | tail -4
AQUA_FUZZ_SEEDS=3 timeout 2400 $CS --tool memcheck python -m pytest tests/test_gpu_mixed_fuzz.py -q -m gpu -p no:cacheprovider > gpurun_out/r02_sanitizer_memcheck_mixed_noleak.log 2>&1; echo "memcheck rc $?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/r02_sanitizer_memcheck_mixed_noleak.log | tail -4
