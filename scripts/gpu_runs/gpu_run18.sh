cd $GRAFT_REPO_ROOT
timeout 600 python scripts/sweep.py torch_baseline > gpurun_out/r01_torch_baseline.jsonl 2>&1; echo "tb $?"; cat gpurun_out/r01_torch_baseline.jsonl
