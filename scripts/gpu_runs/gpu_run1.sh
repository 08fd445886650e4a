cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; lscpu | grep "Model name"
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -40
timeout 400 python bench.py --steps 20 --warmup 3 --cpu-seconds 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
echo "bench exit $?"; tail -c 3000 gpurun_out/bench1.json; tail -20 gpurun_out/bench1.err
