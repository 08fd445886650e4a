cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -3
timeout 900 python scripts/c3_run.py --policy cfs-host --exchange --check-oracle > gpurun_out/r01_c3_host_exchange.json 2>&1; echo "host xchg $?"; python -c "
import json; d=json.load(open('gpurun_out/r01_c3_host_exchange.json')); print(d['streams'], d['oracle_log_equal'], d['verify_mismatches'], d['swap_device_ms'], d['wall_s'], d['responsiveness_model_s'])"
