cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; lscpu | grep "Model name"
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 1200 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -20
timeout 400 python bench.py > gpurun_out/r01_bench_s2.json 2> gpurun_out/bench.err
echo "bench exit $?"; tail -c 4000 gpurun_out/r01_bench_s2.json; tail -5 gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01_bench_ref_s2.json 2>>gpurun_out/bench.err; tail -c 1500 gpurun_out/r01_bench_ref_s2.json
