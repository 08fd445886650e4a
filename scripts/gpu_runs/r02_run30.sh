cd $GRAFT_REPO_ROOT
AQUA_SWEEP_S=512,1024,2048,4096,8192 timeout 900 python scripts/sweep.py small_ldst > gpurun_out/r02_small_device.jsonl 2>gpurun_out/err.log; tail -2 gpurun_out/err.log
python - <<'PY'
import json
for l in open('gpurun_out/r02_small_device.jsonl'):
    r=json.loads(l); print(r['S'], r['engine'], r['cap'], r['kernel'], r['variant'], r['grid'], r['launch'][:26], r['hbm_GBps_queued'], r['hbm_GBps_device_out'], r['hbm_GBps_device_in'])
PY
