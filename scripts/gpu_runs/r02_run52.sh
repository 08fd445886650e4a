cd $GRAFT_REPO_ROOT
for cfg in 256x2 256x4 512x2 128x4 128x8; do
AQUA_SMALL_CFG=$cfg timeout 900 python scripts/sweep.py small_async >> gpurun_out/r02_small_async.jsonl 2>>gpurun_out/err.log
done
python - <<'PY'
import json
for l in open('gpurun_out/r02_small_async.jsonl'):
    r=json.loads(l); print(r['S'], r['cap'], r['engine'], r['cfg'], r['kernel'], r['variant'], r['grid'], r['threads'], r['out_GBps_rw'], r['in_GBps_rw'])
PY
tail -3 gpurun_out/err.log
