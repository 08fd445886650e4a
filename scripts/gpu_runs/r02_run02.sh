cd $GRAFT_REPO_ROOT
free -g | head -2; nproc
timeout 1500 python -m pytest tests/test_gpu_peer.py tests/test_gpu_ipc.py tests/test_gpu_fullsize.py -q -rs --durations=10 2>&1 | tail -30
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
