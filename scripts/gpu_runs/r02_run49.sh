cd $GRAFT_REPO_ROOT
timeout 900 python scripts/sweep.py small_caps > gpurun_out/r02_small_caps.jsonl 2>gpurun_out/err.log; echo "rc $?"
python - <<'PY'
import json
for l in open('gpurun_out/r02_small_caps.jsonl'):
    r=json.loads(l); print(r['S'], r['cap'], r['engine'], r['kernel'], r['variant'], r['grid'], r['threads'], r['out_GBps_rw'], r['in_GBps_rw'], r['per_sm_rw'])
PY
tail -3 gpurun_out/err.log
