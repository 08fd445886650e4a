cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -2
for x in "--native --check-oracle" "--native --exchange --check-oracle"; do
timeout 900 python scripts/c3_run.py --policy cfs-peer $x > gpurun_out/r01_c3_native.json 2>&1; echo "native $x $?"; python -c "
import json; d=json.load(open('gpurun_out/r01_c3_native.json')); print('wall', d['wall_s'], d.get('oracle_log_equal'), d['verify_mismatches'], d['kernel_launches'], d['iterations'])"
done
timeout 900 python scripts/c3_run.py --policy cfs-host --native --exchange > gpurun_out/r01_c3_native_host_x.json 2>&1; echo "native host x $?"; python -c "
import json; d=json.load(open('gpurun_out/r01_c3_native_host_x.json')); print('wall', d['wall_s'], d['verify_mismatches'])"
