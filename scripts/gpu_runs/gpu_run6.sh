cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -4
timeout 400 python bench.py --steps 30 --warmup 5 --no-host-baselines --no-cpu-baseline > gpurun_out/r01_bench_c2.json 2>&1; echo "c2 $?"
python -c "import json; d=json.load(open('gpurun_out/r01_bench_c2.json')); print(d['value'], d['roofline']['achieved'], d['roofline']['swap_in_achieved'], d['preempt_resume_ms']['sum_device_ms'])"
timeout 400 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r01_bench_c4.json 2>&1; echo "c4 $?"
python -c "import json; d=json.load(open('gpurun_out/r01_bench_c4.json')); print(d['value'], d['roofline']['achieved'], d['roofline']['swap_in_achieved'], d['preempt_resume_ms'], d['parity'])"
timeout 600 python scripts/sweep.py stages > gpurun_out/r01_stages2.jsonl 2>&1; echo "stages $?"
timeout 900 python scripts/sweep.py c5 > gpurun_out/r01_c5_self.jsonl 2>&1; echo "c5 $?"
timeout 900 python scripts/sweep.py c5host > gpurun_out/r01_c5_host.jsonl 2>&1; echo "c5host $?"
timeout 600 python scripts/sweep.py host_ctas > gpurun_out/r01_host_ctas.jsonl 2>&1; echo "hostctas $?"
timeout 600 python scripts/sweep.py self_ctas > gpurun_out/r01_self_ctas.jsonl 2>&1; echo "selfctas $?"
cat gpurun_out/r01_host_ctas.jsonl gpurun_out/r01_self_ctas.jsonl
