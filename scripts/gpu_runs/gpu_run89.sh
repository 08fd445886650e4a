cd $GRAFT_REPO_ROOT
K="(test_random_sequences_bytes and (s512 or s1k or s2k) and (tma_hybrid or ldst_claim) and seed0 is not None) or test_block_major or test_auto_policy"
K2="(s512 or s1k or s2k or test_block_major or test_auto_policy) and (tma_hybrid or ldst_claim or tma or block_major or auto)"
timeout 2400 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$K2" > gpurun_out/r01_sanitizer_memcheck_pack.log 2>&1; echo "memcheck $?"; tail -4 gpurun_out/r01_sanitizer_memcheck_pack.log
