cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -4
timeout 900 python scripts/sweep.py duplex > gpurun_out/r01_duplex2.jsonl 2>&1; echo "duplex $?"; cat gpurun_out/r01_duplex2.jsonl
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r01_bench_hostce.json 2>&1; echo "bench $?"; python -c "
import json; d=json.load(open('gpurun_out/r01_bench_hostce.json')); print(json.dumps(d['host_baseline']))"
