cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r02_gpu_suite8.log 2>&1; echo "suite rc $?"; tail -2 gpurun_out/r02_gpu_suite8.log
rm -f gpurun_out/r02_small_chunks_auto_final.jsonl
for bm in 0 1; do
AQUA_SWEEP_BLOCK_MAJOR=$bm AQUA_SWEEP_S=512,1024,2048,4096,8192,32768 AQUA_SWEEP_ENGINES=auto timeout 900 python scripts/sweep.py small_chunks2 >> gpurun_out/r02_small_chunks_auto_final.jsonl 2>>gpurun_out/err.log
done
python - <<'PY'
import json
for l in open('gpurun_out/r02_small_chunks_auto_final.jsonl'):
    r=json.loads(l); print(r['S'], r['block_major'], r['cap'], r['kernel'], r['variant'], r['launch'][:28], r['hbm_GBps'])
PY
