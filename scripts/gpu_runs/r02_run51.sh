cd $GRAFT_REPO_ROOT
for cfg in 256x2 256x4 512x2 128x4 128x8; do
AQUA_SMALL_CFG=$cfg timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "ldst_async" > gpurun_out/r02_async_tests_$cfg.log 2>&1; echo "$cfg tests rc $?"; tail -1 gpurun_out/r02_async_tests_$cfg.log
done
