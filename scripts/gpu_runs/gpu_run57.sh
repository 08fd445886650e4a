cd $GRAFT_REPO_ROOT
AQUA_SWEEP_SCHED="2:0,4:0" AQUA_SWEEP_CTAS=0 AQUA_SWEEP_STAGES="0,3,5,6,8" AQUA_SWEEP_PIECES="16384,24576,32768,65536" timeout 1500 python scripts/sweep.py tma_sched > gpurun_out/r01_tma_pieces.jsonl 2>gpurun_out/err.log; python - <<'PY'
import json
rows=[json.loads(l) for l in open('gpurun_out/r01_tma_pieces.jsonl')]
for shape in ('c2','c4'):
    r=sorted([x for x in rows if x['shape']==shape], key=lambda x:-x['hbm_GBps'])
    for x in r[:8]: print(shape, x['tma_sched'], x['stages'], x['piece'], x['hbm_GBps'], x['out_hbm_GBps'], x['in_hbm_GBps'])
PY
tail -3 gpurun_out/err.log
