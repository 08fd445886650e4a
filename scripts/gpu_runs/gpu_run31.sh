cd $GRAFT_REPO_ROOT
timeout 900 python scripts/sweep.py layer_overlap > gpurun_out/r01_layer_overlap.jsonl 2>&1; echo "lo $?"; cat gpurun_out/r01_layer_overlap.jsonl
