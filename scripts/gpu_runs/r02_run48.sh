cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -Iinclude scripts/host_cost.cu -Lpaper_2407_21255_b200 -laqua -Xlinker -rpath,$PWD/paper_2407_21255_b200 -o /tmp/host_cost && /tmp/host_cost gpu > gpurun_out/r02_host_cost2.jsonl 2>&1; cat gpurun_out/r02_host_cost2.jsonl
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r02_gpu_suite10.log 2>&1; echo "suite rc $?"; tail -2 gpurun_out/r02_gpu_suite10.log
