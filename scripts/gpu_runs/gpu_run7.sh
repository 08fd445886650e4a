cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -4
timeout 300 python scripts/sweep.py migrate > gpurun_out/r01_migrate.jsonl 2>&1; echo "mig $?"; cat gpurun_out/r01_migrate.jsonl
timeout 900 python scripts/c3_run.py --policy cfs-peer --elastic 40,80 --check-oracle > gpurun_out/r01_c3_elastic.json 2> gpurun_out/r01_c3_elastic.err; echo "c3 elastic $?"; cat gpurun_out/r01_c3_elastic.json; tail -n 3 gpurun_out/r01_c3_elastic.err
