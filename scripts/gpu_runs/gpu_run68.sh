cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --extended-lambda -o /tmp/hbm_probe scripts/hbm_probe.cu
timeout 300 /tmp/hbm_probe | tee gpurun_out/r01_hbm_probe2.jsonl
