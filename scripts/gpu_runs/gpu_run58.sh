cd $GRAFT_REPO_ROOT
B="python bench.py --steps 3 --warmup 3 --no-host-baselines --no-cpu-baseline"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_final.csv $B > /dev/null 2>&1; echo "launch list $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:swap_tma_kernel -s 6 -c 2 -o gpurun_out/r01_prof_tma_final2 $B > gpurun_out/ncu_full_final2.log 2>&1; echo "full $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:swap_tma_kernel -s 6 -c 2 -o gpurun_out/r01_prof_tma_c4_final2 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_c4_final2.log 2>&1; echo "full c4 $?"
