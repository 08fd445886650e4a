cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -8
for im in 4064 256; do
timeout 300 python bench.py --inline-max $im --no-host-baselines --no-cpu-baseline > gpurun_out/r01_bench_inline$im.json 2>>gpurun_out/err.log
python -c "import json;d=json.load(open('gpurun_out/r01_bench_inline$im.json'));print($im, d['value'], d['launch_ms'], d['roofline']['achieved'], d['e2e']['value'], d['preempt_resume_ms'])"
done
timeout 600 python scripts/sweep.py latency > gpurun_out/r01_latency_inline.jsonl 2>>gpurun_out/err.log
AQUA_SWEEP_INLINE=256 timeout 600 python scripts/sweep.py latency > gpurun_out/r01_latency_staged.jsonl 2>>gpurun_out/err.log
cat gpurun_out/r01_latency_inline.jsonl gpurun_out/r01_latency_staged.jsonl; tail -5 gpurun_out/err.log
