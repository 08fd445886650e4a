cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -3
timeout 900 python scripts/c3_run.py --policy cfs-peer --check-oracle > gpurun_out/r01_c3_peer2.json 2>&1; echo "c3 $?"; python -c "
import json; d=json.load(open('gpurun_out/r01_c3_peer2.json')); print('wall', d['wall_s'], d['oracle_log_equal'], d['verify_mismatches'], d['swap_GBps'])"
AQUA_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 scripts/sweep.py c5_multi > gpurun_out/r01_c5_multi_shared.jsonl 2> gpurun_out/r01_c5_multi_shared.err; echo "c5multi $?"; head -5 gpurun_out/r01_c5_multi_shared.jsonl; tail -n 3 gpurun_out/r01_c5_multi_shared.err
