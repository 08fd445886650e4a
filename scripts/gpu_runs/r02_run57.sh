cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "exchange" -p no:cacheprovider > gpurun_out/r02_new_tests2.log 2>&1; echo "new tests rc $?"; tail -3 gpurun_out/r02_new_tests2.log
timeout 1200 python scripts/product_mutants.py run --kind gpu --only "exchange: every resume" --timeout 600 --out gpurun_out/r02_product_mutants_gpu_xchg.json > gpurun_out/r02_product_mutants_gpu_xchg.log 2>&1; echo "mutants rc $?"
tail -3 gpurun_out/r02_product_mutants_gpu_xchg.log
