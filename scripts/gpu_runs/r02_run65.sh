cd $GRAFT_REPO_ROOT
timeout 600 python scripts/sweep.py migrate > gpurun_out/r02_migrate.jsonl 2>&1; echo "mig $?"; cat gpurun_out/r02_migrate.jsonl
timeout 900 python scripts/sweep.py prefix > gpurun_out/r02_prefix.jsonl 2>&1; echo "prefix $?"; cat gpurun_out/r02_prefix.jsonl
timeout 900 python scripts/sweep.py layers > gpurun_out/r02_layers.jsonl 2>&1; echo "layers $?"; cat gpurun_out/r02_layers.jsonl
