cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "descriptor_ring" -p no:cacheprovider > gpurun_out/r02_new_tests3.log 2>&1; echo "new tests rc $?"; tail -3 gpurun_out/r02_new_tests3.log
timeout 2400 python scripts/product_mutants.py run --kind gpu --only "descriptor ring" --timeout 600 --out gpurun_out/r02_product_mutants_gpu5.json > gpurun_out/r02_product_mutants_gpu5.log 2>&1; echo "mutants rc $?"
tail -6 gpurun_out/r02_product_mutants_gpu5.log
