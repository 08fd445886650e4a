cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 300 -x 2>&1 | tail -4
timeout 400 python bench.py > gpurun_out/r01_bench_host_fast.json 2> gpurun_out/bench.err; echo "bench exit $?"
python -c "import json;d=json.load(open('gpurun_out/r01_bench_host_fast.json'));print(d['value'], d['roofline']['achieved'], d['roofline']['swap_in_achieved'], d['e2e'], d['preempt_resume_ms'], d['preempt_resume_vs_host'], d['parity'], d['clocks'])"
timeout 600 python scripts/sweep.py latency > gpurun_out/r01_latency_fast.jsonl 2>>gpurun_out/bench.err; cat gpurun_out/r01_latency_fast.jsonl
