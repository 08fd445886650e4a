cd $GRAFT_REPO_ROOT
for pol in fcfs cfs-peer cfs-host; do
timeout 900 python scripts/c3_run.py --policy $pol > gpurun_out/r01_c3_$pol.json 2> gpurun_out/r01_c3_$pol.err; echo "$pol $?"; python -c "
import json; d=json.load(open('gpurun_out/r01_c3_$pol.json')); print(d['policy'], d['responsiveness_model_s'], d.get('per_prompt_ms'), d['verify_mismatches'])"; tail -n 2 gpurun_out/r01_c3_$pol.err
done
