cd $GRAFT_REPO_ROOT
B="python bench.py --steps 3 --warmup 3 --no-host-baselines --no-cpu-baseline"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_s2.csv $B > /dev/null 2>&1; echo "launch list $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:swap_tma_kernel -s 6 -c 2 -o gpurun_out/r01_prof_tma_s2 $B > gpurun_out/ncu_full_s2.log 2>&1; echo "full $?"; tail -3 gpurun_out/ncu_full_s2.log
timeout 600 ncu --metrics gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none -k regex:swap_tma_kernel --csv --log-file gpurun_out/r01_ncu_host_pcie.csv python scripts/sweep.py host_pcie > gpurun_out/host_pcie.log 2>&1; echo "pcie $?"; tail -3 gpurun_out/host_pcie.log; head -c 3000 gpurun_out/r01_ncu_host_pcie.csv
