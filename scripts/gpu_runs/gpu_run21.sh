cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "exchange and host" 2>&1 | grep -E "Error|error|assert|^E " | head -20
