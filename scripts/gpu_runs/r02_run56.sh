cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "delayed_stream or hybrid_register_warps or adversarial or migration_source or staging_shared or prefix_cache_reuse" -p no:cacheprovider > gpurun_out/r02_new_tests.log 2>&1; echo "new tests rc $?"; tail -3 gpurun_out/r02_new_tests.log
timeout 3000 python scripts/product_mutants.py run --kind gpu --timeout 600 --out gpurun_out/r02_product_mutants_gpu.json > gpurun_out/r02_product_mutants_gpu.log 2>&1; echo "mutants rc $?"
tail -17 gpurun_out/r02_product_mutants_gpu.log
