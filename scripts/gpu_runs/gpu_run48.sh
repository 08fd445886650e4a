cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 300 -x 2>&1 | tail -4
timeout 400 python bench.py > gpurun_out/r01_bench_dyn.json 2> gpurun_out/bench.err; echo "bench exit $?"
python -c "import json;d=json.load(open('gpurun_out/r01_bench_dyn.json'));print(d['value'], d['launch_ms'], d['roofline'], d['e2e']['value'], d['preempt_resume_ms']['sum_device_ms'], d['parity'], d['clocks'])"
timeout 300 python bench.py --config c4 --no-host-baselines --no-cpu-baseline > gpurun_out/r01_bench_c4_dyn.json 2>> gpurun_out/bench.err; echo "c4 exit $?"
python -c "import json;d=json.load(open('gpurun_out/r01_bench_c4_dyn.json'));print(d['value'], d['roofline']['achieved'], d['roofline']['swap_in_achieved'], d['parity'])"
timeout 600 python scripts/c3_run.py --policy cfs-peer --check-oracle > gpurun_out/r01_c3_peer_dyn.json 2> gpurun_out/r01_c3_peer_dyn.err; echo "c3 peer exit $?"; tail -c 1500 gpurun_out/r01_c3_peer_dyn.json; tail -3 gpurun_out/r01_c3_peer_dyn.err
