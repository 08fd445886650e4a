cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf --timeout 300 2>&1 | tail -5
timeout 300 python bench.py --no-host-baselines > gpurun_out/r01_bench_rings_check.json 2>gpurun_out/err.log; tail -c 600 gpurun_out/r01_bench_rings_check.json; tail -3 gpurun_out/err.log
