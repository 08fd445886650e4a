cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "fragmented_slots or migrate" -p no:cacheprovider > gpurun_out/r02_migruns.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/r02_migruns.log
timeout 600 python scripts/sweep.py migrate > gpurun_out/r02_migrate_ce2.jsonl 2> gpurun_out/r02_migrate_ce2.err; echo "migrate rc $?"; cat gpurun_out/r02_migrate_ce2.jsonl; tail -2 gpurun_out/r02_migrate_ce2.err
timeout 2400 python scripts/product_mutants.py run --kind gpu --only "migration on the copy engines: a run ignores the destination" --timeout 600 --out gpurun_out/r02_product_mutants_gpu_migce2.json > gpurun_out/r02_product_mutants_gpu_migce2.log 2>&1; echo "mutants rc $?"; tail -3 gpurun_out/r02_product_mutants_gpu_migce2.log
