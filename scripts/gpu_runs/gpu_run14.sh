cd $GRAFT_REPO_ROOT
timeout 600 python scripts/sweep.py ctas_stages > gpurun_out/r01_ctas_stages.jsonl 2>&1; echo "cs $?"; cat gpurun_out/r01_ctas_stages.jsonl
timeout 600 python bench.py --no-cpu-baseline --no-host-baselines > gpurun_out/r01_bench_rich.json 2>&1; echo "bench $?"; python -c "
import json; d=json.load(open('gpurun_out/r01_bench_rich.json')); print(d['launch_ms'], d['launch_shape'], d['host'], d['preempt_resume_ms'])"
