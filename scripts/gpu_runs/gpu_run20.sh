cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -3
timeout 600 python scripts/sweep.py exchange > gpurun_out/r01_exchange.jsonl 2>&1; echo "xchg $?"; cat gpurun_out/r01_exchange.jsonl
