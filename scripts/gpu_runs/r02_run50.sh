cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r02_gpu_suite11.log 2>&1; echo "suite rc $?"; tail -2 gpurun_out/r02_gpu_suite11.log
AQUA_SWEEP_S=512,1024,2048 timeout 900 python scripts/sweep.py small_caps > gpurun_out/r02_small_caps_auto.jsonl 2>gpurun_out/err.log; echo "rc $?"
python - <<'PY'
import json
for l in open('gpurun_out/r02_small_caps_auto.jsonl'):
    r=json.loads(l); print(r['S'], r['cap'], r['engine'], r['kernel'], r['variant'], r['grid'], r['threads'], r['out_GBps_rw'], r['in_GBps_rw'], r['per_sm_rw'])
PY
timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "ldst_small or auto_policy" > gpurun_out/r02_sanitizer_memcheck_small2.log 2>&1; echo "memcheck rc $?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/r02_sanitizer_memcheck_small2.log | tail -3
