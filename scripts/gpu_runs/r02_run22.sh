cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "ldst" > gpurun_out/r02_small_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/r02_small_tests.log
for cps in 2 3 4 6 8; do
AQUA_SMALL_CPS=$cps timeout 900 python scripts/sweep.py small_ldst >> gpurun_out/r02_small_ldst.jsonl 2>>gpurun_out/err.log
done
cat gpurun_out/r02_small_ldst.jsonl; tail -2 gpurun_out/err.log
