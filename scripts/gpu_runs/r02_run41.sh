cd $GRAFT_REPO_ROOT
# one-off long fuzz: 24 seeds x 60 ops per sequence (the suite: 2 x 25), every engine and shape, both grids
AQUA_FUZZ_SEEDS=24 AQUA_FUZZ_OPS=60 timeout 2400 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "random_sequences or multistream_fuzz" > gpurun_out/r02_long_fuzz.log 2>&1; echo "rc $?"; tail -3 gpurun_out/r02_long_fuzz.log
