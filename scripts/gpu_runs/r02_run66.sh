cd $GRAFT_REPO_ROOT
timeout 900 python scripts/c3_run.py --policy cfs-peer --check-oracle > gpurun_out/r02_c3_peer_s4.json 2> gpurun_out/r02_c3.err; echo "c3 rc $?"
timeout 900 python scripts/c3_run.py --policy cfs-peer --native --check-oracle > gpurun_out/r02_c3_peer_native_s4.json 2>> gpurun_out/r02_c3.err; echo "c3 native rc $?"
timeout 900 python scripts/c3_run.py --policy cfs-host --exchange --check-oracle > gpurun_out/r02_c3_host_exchange_s4.json 2>> gpurun_out/r02_c3.err; echo "c3 host rc $?"
python - <<'PY'
import json
for f in ("r02_c3_peer_s4", "r02_c3_peer_native_s4", "r02_c3_host_exchange_s4"):
    d = json.load(open(f"gpurun_out/{f}.json"))
    print(f, d.get("wall_s"), d.get("swap_GBps"), d.get("oracle_log_equal"), d.get("verify_mismatches"), d.get("per_prompt_ms"))
PY
tail -3 gpurun_out/r02_c3.err
