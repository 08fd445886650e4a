cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/r02_bench_s3.json 2>gpurun_out/bench_err.log; echo "bench rc $?"; tail -c 600 gpurun_out/r02_bench_s3.json; tail -3 gpurun_out/bench_err.log
timeout 900 python scripts/sweep.py c5 > gpurun_out/r02_c5_self.jsonl 2>>gpurun_out/err.log; echo "c5 rc $?"
python - <<'PY'
import json
for l in open('gpurun_out/r02_c5_self.jsonl'):
    r=json.loads(l); print(r['bs'], r['blocks'], r['out_GBps'], r['in_GBps'])
PY
