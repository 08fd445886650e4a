cd $GRAFT_REPO_ROOT
timeout 600 python scripts/sweep.py ldst_variants > gpurun_out/r01_ldst_variants.jsonl 2>&1; echo "lv $?"; cat gpurun_out/r01_ldst_variants.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "ldst" 2>&1 | tail -2
