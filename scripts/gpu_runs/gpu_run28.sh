cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -3
for x in "" "--exchange"; do
timeout 900 python scripts/c3_run.py --policy cfs-host $x > gpurun_out/r01_c3_host_ce$x.json 2>&1; echo "host $x $?"; python -c "
import json; d=json.load(open('gpurun_out/r01_c3_host_ce$x.json')); print(d['streams'], d['verify_mismatches'], d['swap_device_ms'], d['swap_GBps'], 'wall', d['wall_s'], d['responsiveness_model_s'], d['per_prompt_ms'])"
done
timeout 600 python bench.py --steps 30 > gpurun_out/r01_bench_final2.json 2>&1; echo "bench $?"; python -c "
import json; d=json.load(open('gpurun_out/r01_bench_final2.json')); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['host_baseline']['best'], d['host_baseline']['best_preempt_resume_ms'], d['clocks'])"
