cd $GRAFT_REPO_ROOT
AQUA_FUZZ_SEEDS=200 AQUA_FUZZ_OPS=80 timeout 2400 python -m pytest tests/test_gpu_mixed_fuzz.py -q -m gpu -x -p no:cacheprovider > gpurun_out/r02_mixed_fuzz_s5.log 2>&1; echo "mixed fuzz rc $?"; tail -2 gpurun_out/r02_mixed_fuzz_s5.log
AQUA_FUZZ_SEEDS=24 AQUA_FUZZ_OPS=60 timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py -q -m gpu -x -k "random_sequences" -p no:cacheprovider > gpurun_out/r02_random_seq_s5.log 2>&1; echo "random seq rc $?"; tail -2 gpurun_out/r02_random_seq_s5.log
