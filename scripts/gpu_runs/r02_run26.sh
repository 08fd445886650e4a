cd $GRAFT_REPO_ROOT
AQUA_SWEEP_BLOCK_MAJOR=1 AQUA_SWEEP_S=512,1024,2048,4096 timeout 900 python scripts/sweep.py small_chunks2 > gpurun_out/r02_small_chunks_bm2.jsonl 2>gpurun_out/err.log; tail -2 gpurun_out/err.log
python - <<'PY'
import json
for l in open('gpurun_out/r02_small_chunks_bm2.jsonl'):
    r=json.loads(l); print(r['S'], r['cap'], r['engine'], r['sched_units'] if r['engine']!='auto' else '-', r['kernel'], r['variant'], r['launch'][:28], r['hbm_GBps'])
PY
