cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/scatter_probe scripts/scatter_probe.cu && timeout 900 /tmp/scatter_probe > gpurun_out/r02_scatter_probe.jsonl 2>&1; echo "rc $?"; cat gpurun_out/r02_scatter_probe.jsonl
