cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-host-baselines --no-cpu-baseline > gpurun_out/r02_bench_e2e.json 2>gpurun_out/bench_err.log; echo "bench rc $?"
timeout 900 python bench.py --config c4 --no-host-baselines --no-cpu-baseline > gpurun_out/r02_bench_c4_e2e.json 2>>gpurun_out/bench_err.log; echo "c4 rc $?"
python - <<'PY'
import json
for f in ("r02_bench_e2e", "r02_bench_c4_e2e"):
    d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    print(f, d["value"], d["e2e"], d["preempt_resume_ms"]["e2e_step_p50_ms"], d["ms_per_step"])
PY
tail -3 gpurun_out/bench_err.log
timeout 900 python -m pytest tests -q -m gpu -k "bench" > gpurun_out/r02_bench_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/r02_bench_tests.log
