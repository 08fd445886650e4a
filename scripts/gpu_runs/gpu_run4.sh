cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -6
timeout 300 python scripts/sweep.py latency > gpurun_out/r01_latency.jsonl 2>&1; echo "lat exit $?"
timeout 600 python scripts/sweep.py stages > gpurun_out/r01_stages.jsonl 2>&1; echo "stages exit $?"
timeout 600 python scripts/c3_run.py --policy cfs-peer --check-oracle > gpurun_out/r01_c3_peer.json 2> gpurun_out/r01_c3_peer.err; echo "c3 peer exit $?"
timeout 900 python scripts/c3_run.py --policy cfs-host > gpurun_out/r01_c3_host.json 2> gpurun_out/r01_c3_host.err; echo "c3 host exit $?"
cat gpurun_out/r01_c3_peer.json gpurun_out/r01_c3_host.json; tail -n 3 gpurun_out/r01_c3_host.err
