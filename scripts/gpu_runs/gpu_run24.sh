cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -3
for pol in cfs-host cfs-peer; do for x in "" "--exchange"; do
timeout 900 python scripts/c3_run.py --policy $pol $x > gpurun_out/r01_c3_$pol$x.json 2>&1; echo "$pol $x $?"; python -c "
import json; d=json.load(open('gpurun_out/r01_c3_$pol$x.json')); print(d['streams'], d['verify_mismatches'], d['swap_device_ms'], 'wall', d['wall_s'], 'model', d['responsiveness_model_s']['makespan'], d['responsiveness_model_s']['tpot_p99'])"
done; done
