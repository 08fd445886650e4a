cd $GRAFT_REPO_ROOT
free -g | head -2
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -15
timeout 400 python bench.py --steps 30 --warmup 5 --cpu-seconds 10 > gpurun_out/r01_bench2.json 2> gpurun_out/r01_bench2.err; echo "bench exit $?"; tail -c 1500 gpurun_out/r01_bench2.json; tail -5 gpurun_out/r01_bench2.err
timeout 300 python scripts/sweep.py latency > gpurun_out/r01_latency.jsonl 2>&1; echo "lat exit $?"
timeout 600 python scripts/c3_run.py --policy cfs-peer --check-oracle > gpurun_out/r01_c3_peer.json 2> gpurun_out/r01_c3_peer.err; echo "c3 peer exit $?"
timeout 900 python scripts/c3_run.py --policy cfs-host > gpurun_out/r01_c3_host.json 2> gpurun_out/r01_c3_host.err; echo "c3 host exit $?"
timeout 600 python scripts/c3_run.py --policy fcfs > gpurun_out/r01_c3_fcfs.json 2> gpurun_out/r01_c3_fcfs.err; echo "c3 fcfs exit $?"
cat gpurun_out/r01_c3_*.json; tail -3 gpurun_out/r01_c3_*.err
