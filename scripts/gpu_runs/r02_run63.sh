cd $GRAFT_REPO_ROOT
AQUA_SWEEP_S=512,1024 timeout 600 python scripts/sweep.py block_order > gpurun_out/r02_block_order_ring1m.jsonl 2>&1; echo "rc $?"; cat gpurun_out/r02_block_order_ring1m.jsonl
AQUA_STAGE_MIN_BYTES=67108864 AQUA_SWEEP_S=512,1024 timeout 600 python scripts/sweep.py block_order > gpurun_out/r02_block_order_ring64m.jsonl 2>&1; echo "rc $?"; cat gpurun_out/r02_block_order_ring64m.jsonl
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -Iinclude scripts/host_cost.cu -Lpaper_2407_21255_b200 -laqua -Xlinker -rpath,$PWD/paper_2407_21255_b200 -o /tmp/host_cost && /tmp/host_cost gpu | tail -3
