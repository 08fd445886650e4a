cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "ldst_small" > gpurun_out/r02_small_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/r02_small_tests.log
for cps in 1 2 3 4 8; do
AQUA_SMALL_CPS=$cps timeout 900 python scripts/sweep.py small_ldst >> gpurun_out/r02_small_ldst2.jsonl 2>>gpurun_out/err.log
done
grep small gpurun_out/r02_small_ldst2.jsonl | cut -c1-150; tail -2 gpurun_out/err.log
