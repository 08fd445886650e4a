cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 300 -x 2>&1 | tail -3
timeout 400 python bench.py > gpurun_out/r01_bench_final3.json 2> gpurun_out/bench.err; echo "bench exit $?"
python -c "import json;d=json.load(open('gpurun_out/r01_bench_final3.json'));print(d['value'], d['roofline'], d['e2e']['value'], d['preempt_resume_ms']['sum_device_ms'], d['preempt_resume_vs_host'], d['parity'], d['clocks'], d['cpu_baseline'])"
