cd $GRAFT_REPO_ROOT
AQUA_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 scripts/c3_tp.py > gpurun_out/r01_c3_tp2_shared.json 2> gpurun_out/r01_c3_tp2_shared.err; echo "tp $?"; cat gpurun_out/r01_c3_tp2_shared.json; tail -n 3 gpurun_out/r01_c3_tp2_shared.err
