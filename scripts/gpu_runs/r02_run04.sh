cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_peer.py tests/test_gpu_ipc.py -q -rs > gpurun_out/r02_new_tests2.log 2>&1; echo "new rc $?"; tail -3 gpurun_out/r02_new_tests2.log
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r02_gpu_suite.log 2>&1; echo "suite rc $?"; tail -3 gpurun_out/r02_gpu_suite.log
python scripts/nvlink_peer.py
AQUA_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 scripts/nvlink_interference.py --ctas 0,16 --weights-gb 4 > gpurun_out/r02_interference_shared_smoke.jsonl 2> gpurun_out/r02_interference_shared_smoke.err; echo "interf rc $?"; cat gpurun_out/r02_interference_shared_smoke.jsonl
timeout 600 python bench.py > gpurun_out/r02_bench1.json 2> gpurun_out/r02_bench1.err; echo "bench rc $?"; head -c 600 gpurun_out/r02_bench1.json
