cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_peer.py tests/test_gpu_ipc.py tests/test_gpu_fullsize.py -q -rs --durations=10 > gpurun_out/r02_new_tests.log 2>&1; echo "rc $?"
tail -5 gpurun_out/r02_new_tests.log
