cd $GRAFT_REPO_ROOT
timeout 900 python scripts/sweep.py c5 > gpurun_out/r01_c5_self_b2s4.jsonl 2>gpurun_out/err.log; echo "c5 $?"
timeout 900 python scripts/interference.py > gpurun_out/r01_interference3.jsonl 2>&1; echo "interf $?"; cat gpurun_out/r01_interference3.jsonl | cut -c1-300
