cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -3
timeout 600 python scripts/sweep.py self_ctas > gpurun_out/r01_self_ctas_auto.jsonl 2>&1; echo "selfctas $?"; cat gpurun_out/r01_self_ctas_auto.jsonl
timeout 900 python scripts/interference.py > gpurun_out/r01_interference2.jsonl 2>&1; echo "interf $?"; grep equal gpurun_out/r01_interference2.jsonl
timeout 600 python bench.py --no-cpu-baseline --no-host-baselines > gpurun_out/r01_bench_auto.json 2>&1; echo "bench $?"; python -c "
import json; d=json.load(open('gpurun_out/r01_bench_auto.json')); print(d['value'], d['roofline']['achieved'], d['roofline']['swap_in_achieved'], d['launch_ms'])"
timeout 600 python bench.py --config c4 --no-cpu-baseline --no-host-baselines > gpurun_out/r01_bench_c4_auto.json 2>&1; echo "c4 $?"; python -c "
import json; d=json.load(open('gpurun_out/r01_bench_c4_auto.json')); print(d['value'], d['roofline']['achieved'], d['roofline']['swap_in_achieved'])"
