cd $GRAFT_REPO_ROOT
for sd in 2 3 4 5 6; do
timeout 900 python scripts/c3_run.py --policy cfs-peer --check-oracle --trace-seed $sd > gpurun_out/r01_c3_seed$sd.json 2> gpurun_out/c3s.err; echo "seed $sd exit $?"; python -c "import json;d=json.load(open('gpurun_out/r01_c3_seed$sd.json'));print(d['config'][:60], d['swap_out_calls'], d['swap_in_calls'], d['swap_GBps'], d['verify_mismatches'], d['oracle_log_equal'], d['oracle_calls'])"; tail -1 gpurun_out/c3s.err
done
