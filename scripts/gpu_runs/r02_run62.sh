cd $GRAFT_REPO_ROOT
timeout 1200 python scripts/sweep.py block_order > gpurun_out/r02_block_order.jsonl 2> gpurun_out/r02_block_order.err; echo "rc $?"; cat gpurun_out/r02_block_order.jsonl; tail -3 gpurun_out/r02_block_order.err
