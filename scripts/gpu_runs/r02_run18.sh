cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_peer.py -q -m gpu -x > gpurun_out/r02_peer_tests.log 2>&1; echo "peer rc $?"; tail -3 gpurun_out/r02_peer_tests.log
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r02_gpu_suite5.log 2>&1; echo "suite rc $?"; tail -3 gpurun_out/r02_gpu_suite5.log
