cd $GRAFT_REPO_ROOT
timeout 3300 python scripts/product_mutants.py run --kind gpu --only "AUTO:" --timeout 600 --out gpurun_out/r02_product_mutants_gpu_auto.json > gpurun_out/r02_product_mutants_gpu_auto.log 2>&1; echo "mutants rc $?"
tail -32 gpurun_out/r02_product_mutants_gpu_auto.log
