cd $GRAFT_REPO_ROOT
timeout 600 python scripts/nvlink_peer.py --lender 0 --config c2 --ctas 32,0 --steps 3 > gpurun_out/r02_nvlink_peer_smoke.jsonl 2>&1; echo "peer smoke rc $?"; cut -c1-300 gpurun_out/r02_nvlink_peer_smoke.jsonl
timeout 600 python scripts/nvlink_peer.py --lender 0 --config c4 --ctas 0 --steps 3 --bidir > gpurun_out/r02_nvlink_peer_smoke_bidir.jsonl 2>&1; echo "bidir smoke rc $?"; cut -c1-200 gpurun_out/r02_nvlink_peer_smoke_bidir.jsonl
timeout 900 ncu --replay-mode application --clock-control none -k regex:swap_ -c 4 \
  --metrics gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --csv --log-file gpurun_out/r02_nvlink_ncu_smoke.csv \
  python scripts/nvlink_peer.py --lender 0 --config c2 --ctas 32 --steps 1 --warmup 1 > gpurun_out/r02_nvlink_ncu_smoke.log 2>&1; echo "ncu smoke rc $?"; tail -3 gpurun_out/r02_nvlink_ncu_smoke.log; grep -c nvltx gpurun_out/r02_nvlink_ncu_smoke.csv; grep nvltx gpurun_out/r02_nvlink_ncu_smoke.csv | head -2
