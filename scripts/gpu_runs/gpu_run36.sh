cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf --timeout 300 -k "random_sequences" 2>&1 | tail -5
timeout 400 python bench.py > gpurun_out/r01_bench_e2e.json 2> gpurun_out/bench_err.log; tail -3 gpurun_out/bench_err.log
timeout 400 python bench.py --config c4 --no-host-baselines > gpurun_out/r01_bench_c4_e2e.json 2>> gpurun_out/bench_err.log
python - <<'P'
import json
for f in ("gpurun_out/r01_bench_e2e.json", "gpurun_out/r01_bench_c4_e2e.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["value"], d["e2e"], d["roofline"]["frac"], d["clocks"])
P
