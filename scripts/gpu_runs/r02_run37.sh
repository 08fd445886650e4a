cd $GRAFT_REPO_ROOT
timeout 900 python scripts/sweep.py c5 > gpurun_out/r02_c5_self.jsonl 2>>gpurun_out/err.log; echo "c5 rc $?"
python - <<'PY'
import json
for l in open('gpurun_out/r02_c5_self.jsonl'):
    r=json.loads(l); print(r['bs'], r['blocks'], r['out_GBps'], r['in_GBps'])
PY
AQUA_SWEEP_S=512,1024,2048,4096,8192 timeout 900 python scripts/sweep.py small_ldst > gpurun_out/r02_small_device2.jsonl 2>>gpurun_out/err.log
python - <<'PY'
import json
for l in open('gpurun_out/r02_small_device2.jsonl'):
    r=json.loads(l); print(r['S'], r['engine'], r['cap'], r['kernel'], r['variant'], r['grid'], r['hbm_GBps_queued'], r['hbm_GBps_device_out'], r['hbm_GBps_device_in'])
PY
tail -3 gpurun_out/err.log
