cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "exchange" 2>&1 | tail -2
timeout 900 python scripts/sweep.py duplex > gpurun_out/r01_duplex.jsonl 2>&1; echo "duplex $?"; cat gpurun_out/r01_duplex.jsonl
