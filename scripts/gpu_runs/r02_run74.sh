cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "degenerate_and_maximum" -p no:cacheprovider > gpurun_out/r02_edge_tests.log 2>&1; echo "edge rc $?"; tail -15 gpurun_out/r02_edge_tests.log
