cd $GRAFT_REPO_ROOT
K="test_random_sequences_bytes and (tma_dyn1 or tma_hybrid or tma_hyb) and tiny_256B or test_dynamic_schedule_counter or (test_swap_exchange_bytes and lender_dyn and 3)"
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$K" > gpurun_out/r01_sanitizer_memcheck_dyn.log 2>&1; echo "memcheck $?"; tail -5 gpurun_out/r01_sanitizer_memcheck_dyn.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$K" > gpurun_out/r01_sanitizer_racecheck_dyn.log 2>&1; echo "racecheck $?"; tail -5 gpurun_out/r01_sanitizer_racecheck_dyn.log
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$K" > gpurun_out/r01_sanitizer_synccheck_dyn.log 2>&1; echo "synccheck $?"; tail -5 gpurun_out/r01_sanitizer_synccheck_dyn.log
