cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r02_gpu_suite7.log 2>&1; echo "suite rc $?"; tail -2 gpurun_out/r02_gpu_suite7.log
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="(test_random_sequences_bytes and (ldst_small or auto) and (s512 or s1k or s2k or fp8 or s512 or c4_shape)) or (test_block_major_layout_bytes and (ldst_small or auto)) or test_auto_policy"
timeout 1500 $CS --tool memcheck --print-limit 100000 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "$SEL" -p no:cacheprovider > gpurun_out/r02_sanitizer_memcheck_small.log 2>&1; echo "memcheck rc $?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/r02_sanitizer_memcheck_small.log | tail -3
timeout 1500 $CS --tool racecheck python -m pytest tests/test_gpu_parity.py -q -m gpu -k "$SEL" -p no:cacheprovider > gpurun_out/r02_sanitizer_racecheck_small.log 2>&1; echo "racecheck rc $?"; grep -E "RACECHECK SUMMARY|passed|failed" gpurun_out/r02_sanitizer_racecheck_small.log | tail -3
for bm in 0 1; do
AQUA_SWEEP_BLOCK_MAJOR=$bm AQUA_SWEEP_S=512,1024,2048,4096,8192,32768 AQUA_SWEEP_ENGINES=auto timeout 900 python scripts/sweep.py small_chunks2 >> gpurun_out/r02_small_chunks_auto_final.jsonl 2>>gpurun_out/err.log
done
python - <<'PY'
import json
for l in open('gpurun_out/r02_small_chunks_auto_final.jsonl'):
    r=json.loads(l); print(r['S'], r['block_major'], r['cap'], r['kernel'], r['variant'], r['launch'][:28], r['hbm_GBps'])
PY
