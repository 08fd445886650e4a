cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 300 -x 2>&1 | tail -3
timeout 400 python bench.py > gpurun_out/r01_bench_b2s4.json 2> gpurun_out/bench.err; echo "bench exit $?"
python -c "import json;d=json.load(open('gpurun_out/r01_bench_b2s4.json'));print(d['value'], d['roofline']['achieved'], d['roofline']['swap_in_achieved'], d['e2e']['value'], d['preempt_resume_ms']['sum_device_ms'], d['parity'], d['clocks'])"
timeout 300 python bench.py --config c4 --no-host-baselines --no-cpu-baseline > gpurun_out/r01_bench_c4_b2s4.json 2>> gpurun_out/bench.err; echo "c4 exit $?"
python -c "import json;d=json.load(open('gpurun_out/r01_bench_c4_b2s4.json'));print(d['value'], d['roofline']['achieved'], d['roofline']['swap_in_achieved'], d['parity'])"
timeout 600 python scripts/c3_run.py --policy cfs-peer --check-oracle > gpurun_out/r01_c3_peer_b2s4.json 2> gpurun_out/c3.err; echo "c3 exit $?"; python -c "import json;d=json.load(open('gpurun_out/r01_c3_peer_b2s4.json'));print(d['swap_GBps'], d['verify_mismatches'], d['oracle_log_equal'], d['per_prompt_ms'])"
