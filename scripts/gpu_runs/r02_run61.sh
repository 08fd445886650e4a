cd $GRAFT_REPO_ROOT
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="delayed_stream or hybrid_register_warps or migration_source or staging_shared or prefix_cache_reuse or exchange_resume or descriptor_ring"
timeout 1500 $CS --tool racecheck python -m pytest tests/test_gpu_parity.py -q -m gpu -k "$SEL" -p no:cacheprovider > gpurun_out/r02_sanitizer_racecheck_final.log 2>&1; echo "racecheck rc $?"; grep -E "RACECHECK SUMMARY|ERROR SUMMARY|passed|failed" gpurun_out/r02_sanitizer_racecheck_final.log | tail -4
timeout 1500 $CS --tool synccheck python -m pytest tests/test_gpu_parity.py -q -m gpu -k "$SEL" -p no:cacheprovider > gpurun_out/r02_sanitizer_synccheck_final.log 2>&1; echo "synccheck rc $?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/r02_sanitizer_synccheck_final.log | tail -4
AQUA_FUZZ_SEEDS=200 AQUA_FUZZ_OPS=80 timeout 2400 python -m pytest tests/test_gpu_mixed_fuzz.py -q -m gpu -p no:cacheprovider > gpurun_out/r02_mixed_fuzz_final.log 2>&1; echo "mixed fuzz rc $?"; tail -2 gpurun_out/r02_mixed_fuzz_final.log
