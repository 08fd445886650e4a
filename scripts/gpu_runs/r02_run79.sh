cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py tests/test_gpu_mixed_fuzz.py -q -m gpu -p no:cacheprovider > gpurun_out/r02_parity_migce.log 2>&1; echo "parity rc $?"; tail -3 gpurun_out/r02_parity_migce.log
timeout 600 python scripts/sweep.py migrate > gpurun_out/r02_migrate_ce.jsonl 2> gpurun_out/r02_migrate_ce.err; echo "migrate rc $?"; cat gpurun_out/r02_migrate_ce.jsonl; tail -2 gpurun_out/r02_migrate_ce.err
timeout 2400 python scripts/product_mutants.py run --kind gpu --only "migration on the copy engines" --timeout 600 --out gpurun_out/r02_product_mutants_gpu_migce.json > gpurun_out/r02_product_mutants_gpu_migce.log 2>&1; echo "mutants rc $?"; tail -6 gpurun_out/r02_product_mutants_gpu_migce.log
