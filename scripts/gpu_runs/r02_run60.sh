cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke_final.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/r02_smoke_final.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_gpu_suite_final.log 2>&1; echo "gpu suite rc $?"; tail -2 gpurun_out/r02_gpu_suite_final.log
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --leak-check full python -m pytest tests/test_gpu_parity.py -q -m gpu -k "delayed_stream or hybrid_register_warps or migration_source or staging_shared or prefix_cache_reuse or exchange_resume or descriptor_ring or capacity" -p no:cacheprovider > gpurun_out/r02_sanitizer_memcheck_final.log 2>&1; echo "memcheck rc $?"; grep -E "ERROR SUMMARY|LEAK SUMMARY|passed|failed" gpurun_out/r02_sanitizer_memcheck_final.log | tail -4
timeout 600 python bench.py > gpurun_out/r02_bench_final3.json 2> gpurun_out/r02_bench_final3.err; echo "bench rc $?"
timeout 600 python bench.py --config c4 > gpurun_out/r02_bench_c4_final3.json 2>> gpurun_out/r02_bench_final3.err; echo "bench c4 rc $?"
timeout 600 python bench.py --impl reference > gpurun_out/r02_bench_ref_final3.json 2>> gpurun_out/r02_bench_final3.err; echo "ref rc $?"
python - <<'PY'
import json
for f in ("r02_bench_final3", "r02_bench_c4_final3", "r02_bench_ref_final3"):
    d = json.load(open(f"gpurun_out/{f}.json"))
    print(f, d["value"], d.get("e2e", {}).get("value"), (d.get("roofline") or {}).get("frac"), d.get("clocks"))
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_final.csv python bench.py --steps 2 --warmup 3 --no-host-baselines --no-cpu-baseline > gpurun_out/r02_launches_final_bench.log 2>&1; echo "launches rc $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:swap_tma -s 8 -c 2 -o gpurun_out/r02_prof_c2_final python bench.py --steps 2 --warmup 3 --no-host-baselines --no-cpu-baseline > gpurun_out/r02_prof_c2_final.log 2>&1; echo "prof c2 rc $?"
ls -la gpurun_out/*.ncu-rep
