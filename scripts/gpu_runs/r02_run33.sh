cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -Iinclude scripts/host_cost.cu -Lpaper_2407_21255_b200 -laqua -Xlinker -rpath,$PWD/paper_2407_21255_b200 -o /tmp/host_cost && (/tmp/host_cost gpu; /tmp/host_cost dry) > gpurun_out/r02_host_cost.jsonl 2>&1; echo "rc $?"; cat gpurun_out/r02_host_cost.jsonl
