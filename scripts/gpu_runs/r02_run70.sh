cd $GRAFT_REPO_ROOT
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="(test_c1_bytes and (ldst or per_chunk or gather_temp)) or (test_random_sequences_bytes and seed0 and (ldst or ldst_small)) or (test_block_major_layout_bytes and ldst)"
timeout 1800 $CS --tool initcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "$SEL" -p no:cacheprovider > gpurun_out/r02_sanitizer_initcheck_ldst.log 2>&1; echo "initcheck rc $?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/r02_sanitizer_initcheck_ldst.log | tail -3
