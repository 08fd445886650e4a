cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline --no-host-baselines > gpurun_out/r01_bench_refactor.json 2>&1; echo "bench $?"; python -c "
import json; d=json.load(open('gpurun_out/r01_bench_refactor.json')); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['parity'])"
