cd $GRAFT_REPO_ROOT
# small-chunk kernel: pipeline depth (1 / 2 register sets) x CTAs per SM (launch bounds), 512 B .. 2 KiB
for cfg in "1 2" "1 3" "1 4" "2 1" "2 2"; do
set -- $cfg
AQUA_SMALL_PIPE=$1 AQUA_SMALL_CPS=$2 AQUA_SWEEP_S=512,1024,2048 timeout 600 python scripts/sweep.py small_ldst 2>>gpurun_out/err.log | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l)
    if r['engine']=='small' and r['cap']==0:
        r['pipe']=$1; r['cps']=$2; print(json.dumps(r))" >> gpurun_out/r02_small_pipe.jsonl
done
cut -c1-300 gpurun_out/r02_small_pipe.jsonl; tail -2 gpurun_out/err.log
