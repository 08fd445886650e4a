# NVLink recipe for a box with >= 2 GPUs (NVLink GB/s vs 900 from ncu).
# One process drives both GPUs (never wrap a multi-rank command in ncu).  The
# NVLink counters are device-wide, so application replay re-runs the whole
# (deterministic) script once per pass.
cd $GRAFT_REPO_ROOT
NGPU=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > gpurun_out/r02_topo.txt 2>&1
# the parity suite: with >= 2 GPUs the 36 peer cases (lender on GPU 1) run instead of skipping
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r02_gpu_suite_2gpu.log 2>&1; tail -2 gpurun_out/r02_gpu_suite_2gpu.log
timeout 900 python scripts/nvlink_peer.py --config c2 --ctas 8,16,24,32,48,64,0 > gpurun_out/r02_nvlink_peer_c2.jsonl
timeout 900 python scripts/nvlink_peer.py --config c4 --ctas 16,32,64,0 > gpurun_out/r02_nvlink_peer_c4.jsonl
timeout 900 python scripts/nvlink_peer.py --config c2 --ctas 32,0 --bidir > gpurun_out/r02_nvlink_peer_bidir.jsonl
timeout 1800 ncu --replay-mode application --clock-control none -k regex:swap_ -c 4 \
  --metrics gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --csv --log-file gpurun_out/r02_nvlink_ncu.csv \
  python scripts/nvlink_peer.py --config c2 --ctas 32 --steps 1 --warmup 1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  scripts/nvlink_interference.py > gpurun_out/r02_nvlink_interference.jsonl
for n in 2 4 8; do
  [ "$n" -le "$NGPU" ] || continue
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n \
    bench.py --gpus $n --steps 20 --warmup 3 > gpurun_out/r02_bench_n$n.json
done
[ "$NGPU" -ge 8 ] && timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
  --master-port 29530 bench.py --gpus 8 --config c4 --roles split --steps 20 --warmup 3 > gpurun_out/r02_bench_c4_split.json
# C3 with the lender in another process on GPU 1 (IPC over NVLink), call log checked against the oracle
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29540 \
  scripts/c3_run.py --policy cfs-peer --check-oracle > gpurun_out/r02_c3_peer_nvlink.json
