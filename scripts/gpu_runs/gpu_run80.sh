cd $GRAFT_REPO_ROOT
for m in engines migrate prefix layers torch_baseline duplex self_ctas host_ctas; do
  timeout 400 python scripts/sweep.py $m > gpurun_out/chk_$m.jsonl 2> gpurun_out/chk_$m.err; echo "$m exit $? lines $(wc -l < gpurun_out/chk_$m.jsonl)"; tail -1 gpurun_out/chk_$m.err | cut -c1-200
done
AQUA_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 scripts/c3_tp.py > gpurun_out/chk_tp.json 2> gpurun_out/chk_tp.err; echo "tp $?"; head -c 300 gpurun_out/chk_tp.json; tail -1 gpurun_out/chk_tp.err
