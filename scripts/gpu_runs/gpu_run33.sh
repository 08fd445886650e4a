cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -2
timeout 600 python scripts/sweep.py ldst_variants > gpurun_out/r01_ldst_variants2.jsonl 2>&1; echo "lv $?"; cat gpurun_out/r01_ldst_variants2.jsonl
