cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ipc.py -m gpu -q -rf --timeout 600 2>&1 | tail -3
