cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_gpu_suite_ring16.log 2>&1; echo "gpu suite rc $?"; tail -2 gpurun_out/r02_gpu_suite_ring16.log
AQUA_SWEEP_S=512,1024,2048,8192 timeout 600 python scripts/sweep.py block_order > gpurun_out/r02_block_order_ring16m.jsonl 2>&1; echo "rc $?"; cat gpurun_out/r02_block_order_ring16m.jsonl
AQUA_SWEEP_S=512,1024,2048,4096,8192,32768 AQUA_SWEEP_ENGINES=auto timeout 900 python scripts/sweep.py small_chunks2 > gpurun_out/r02_small_chunks_auto_ring16.jsonl 2>&1; echo "rc $?"; cat gpurun_out/r02_small_chunks_auto_ring16.jsonl
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -Iinclude scripts/host_cost.cu -Lpaper_2407_21255_b200 -laqua -Xlinker -rpath,$PWD/paper_2407_21255_b200 -o /tmp/host_cost && /tmp/host_cost gpu > gpurun_out/r02_host_cost3.jsonl; tail -4 gpurun_out/r02_host_cost3.jsonl
timeout 600 python bench.py > gpurun_out/r02_bench_ring16.json 2>/dev/null; echo "bench rc $?"; python -c "import json; d=json.load(open('gpurun_out/r02_bench_ring16.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'])"
