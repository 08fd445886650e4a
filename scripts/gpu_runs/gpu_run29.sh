cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -3
timeout 900 python scripts/c3_run.py --policy cfs-peer --check-oracle > gpurun_out/r01_c3_peer_batchfill.json 2>&1; echo "c3 $?"; python -c "
import json; d=json.load(open('gpurun_out/r01_c3_peer_batchfill.json')); print('wall', d['wall_s'], d['oracle_log_equal'], d['verify_mismatches'], d['kernel_launches'], d['swap_GBps'])"
