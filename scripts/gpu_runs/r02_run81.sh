cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke_s5b.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/r02_smoke_s5b.log
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_gpu_suite_s5b.log 2>&1; echo "gpu suite rc $?"; tail -2 gpurun_out/r02_gpu_suite_s5b.log
for i in 1 2 3; do timeout 600 python bench.py > gpurun_out/r02_bench_s5b$i.json 2>/dev/null; echo "bench $i rc $?"; done
timeout 600 python bench.py --config c4 > gpurun_out/r02_bench_c4_s5b.json 2>/dev/null; echo "c4 rc $?"
timeout 600 python bench.py --impl reference > gpurun_out/r02_bench_ref_s5b.json 2>/dev/null; echo "ref rc $?"
python - <<'PY'
import json
for f in ("r02_bench_s5b1", "r02_bench_s5b2", "r02_bench_s5b3", "r02_bench_c4_s5b", "r02_bench_ref_s5b"):
    d = json.load(open(f"gpurun_out/{f}.json"))
    print(f, d["value"], d.get("e2e", {}).get("value"), (d.get("roofline") or {}).get("frac"), d.get("clocks"), d.get("gpu_launches"))
PY
