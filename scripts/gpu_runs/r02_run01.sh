cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "host_engines or host_staging or c1_bytes or layerwise" 2>&1 | tail -5
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --leak-check full python -m pytest tests/test_gpu_parity.py -x -q -k "host_engines or host_staging" > gpurun_out/r02_memcheck_ce.log 2>&1; echo "memcheck exit $?"; tail -5 gpurun_out/r02_memcheck_ce.log
