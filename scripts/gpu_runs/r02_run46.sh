cd $GRAFT_REPO_ROOT
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/r02_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_final2.json 2>gpurun_out/bench_err.log; echo "bench rc $?"
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_reference2.json 2>>gpurun_out/bench_err.log; echo "ref rc $?"
timeout 900 python bench.py --config c4 --no-host-baselines > gpurun_out/r02_bench_c4_final2.json 2>>gpurun_out/bench_err.log; echo "c4 rc $?"
python - <<'PY'
import json
for f in ("r02_bench_final2", "r02_bench_reference2", "r02_bench_c4_final2"):
    d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    print(f, d["value"], d.get("e2e", {}).get("value"), (d.get("roofline") or {}).get("achieved"), (d.get("roofline") or {}).get("frac"), d.get("clocks"), d.get("gpu_launches"))
PY
tail -3 gpurun_out/bench_err.log
