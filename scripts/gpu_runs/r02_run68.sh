cd $GRAFT_REPO_ROOT
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="test_c1_bytes or (test_random_sequences_bytes and seed0 and (s512 or c4_shape or ragged_10KiB or llama_bs32)) or test_swap_exchange_bytes or test_prefix_cache_bytes or test_migrate_reclaim_relend_bytes"
timeout 1800 $CS --tool initcheck python -m pytest tests/test_gpu_parity.py -q -m gpu -k "$SEL" -p no:cacheprovider > gpurun_out/r02_sanitizer_initcheck.log 2>&1; echo "initcheck rc $?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/r02_sanitizer_initcheck.log | tail -3
grep -B2 -A12 "Uninitialized" gpurun_out/r02_sanitizer_initcheck.log | head -60
