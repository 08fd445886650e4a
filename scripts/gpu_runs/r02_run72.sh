cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "zero_copy_host" -p no:cacheprovider > gpurun_out/r02_new_tests4.log 2>&1; echo "new tests rc $?"; tail -3 gpurun_out/r02_new_tests4.log
timeout 2400 python scripts/product_mutants.py run --kind gpu --only "host-only launches are not capped" --timeout 600 --out gpurun_out/r02_product_mutants_gpu_hostcap.json > gpurun_out/r02_product_mutants_gpu_hostcap.log 2>&1; echo "mutants rc $?"; tail -3 gpurun_out/r02_product_mutants_gpu_hostcap.log
