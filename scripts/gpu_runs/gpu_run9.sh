cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -4
timeout 900 python scripts/sweep.py layers > gpurun_out/r01_layers.jsonl 2>&1; echo "layers $?"; cat gpurun_out/r01_layers.jsonl
timeout 900 python scripts/interference.py > gpurun_out/r01_interference.jsonl 2>&1; echo "interf $?"; cat gpurun_out/r01_interference.jsonl
