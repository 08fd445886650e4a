cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 300 -x 2>&1 | tail -3
timeout 900 python scripts/sweep.py hybrid > gpurun_out/r01_hybrid2.jsonl 2>gpurun_out/err.log; grep '"auto"' gpurun_out/r01_hybrid2.jsonl; tail -3 gpurun_out/err.log
timeout 300 python bench.py --config c4 --max-ctas 32 --no-host-baselines --no-cpu-baseline > gpurun_out/r01_bench_c4_cap32.json 2>>gpurun_out/err.log; python -c "import json;d=json.load(open('gpurun_out/r01_bench_c4_cap32.json'));print(d['value'], d['roofline']['achieved'], d['roofline']['swap_in_achieved'], d['parity'])"
