cd $GRAFT_REPO_ROOT
timeout 400 python bench.py > gpurun_out/r01_bench_final_round.json 2> gpurun_out/bench.err; echo "bench exit $?"
python -c "import json;d=json.load(open('gpurun_out/r01_bench_final_round.json'));print(d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['e2e']['value'], d['preempt_resume_ms']['per_prompt_sum_device_ms'], d['preempt_resume_vs_host'], d['clocks'])"
timeout 300 python bench.py --config c4 --no-host-baselines --no-cpu-baseline > gpurun_out/r01_bench_c4_final_round.json 2>>gpurun_out/bench.err; python -c "import json;d=json.load(open('gpurun_out/r01_bench_c4_final_round.json'));print('c4', d['value'], d['roofline']['achieved'], d['roofline']['traffic'], d['preempt_resume_ms']['per_prompt_sum_device_ms'], d['parity'])"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01_bench_ref_final_round.json 2>>gpurun_out/bench.err; echo "ref $?"
