cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf --timeout 300 -x -k "multistream_fuzz" 2>&1 | tail -3
