cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r02_gpu_suite6.log 2>&1; echo "suite rc $?"; tail -3 gpurun_out/r02_gpu_suite6.log
AQUA_SWEEP_S=512,1024,2048,4096,8192,32768 AQUA_SWEEP_ENGINES=auto timeout 900 python scripts/sweep.py small_chunks2 > gpurun_out/r02_small_chunks_auto2.jsonl 2>gpurun_out/err.log; cut -c1-220 gpurun_out/r02_small_chunks_auto2.jsonl; tail -2 gpurun_out/err.log
timeout 900 python bench.py --no-host-baselines --no-cpu-baseline > gpurun_out/r02_bench4.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/r02_bench4.json'));print(d['value'], d['roofline']['achieved'], d['roofline']['swap_in_achieved'])"
