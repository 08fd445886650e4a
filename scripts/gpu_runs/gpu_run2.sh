cd $GRAFT_REPO_ROOT
B="python bench.py --steps 3 --warmup 3 --no-host-baselines --no-cpu-baseline"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv $B > gpurun_out/ncu_launch_bench.json 2>&1
echo "launch list exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:swap_tma_kernel -s 6 -c 2 -o gpurun_out/r01_prof_tma $B > gpurun_out/ncu_full.log 2>&1
echo "full exit $?"; tail -5 gpurun_out/ncu_full.log
timeout 600 python scripts/sweep.py engines > gpurun_out/r01_sweep_engines.jsonl 2>&1; echo "sweep exit $?"
timeout 900 python scripts/sweep.py c5 > gpurun_out/r01_c5_self.jsonl 2>&1; echo "c5 exit $?"
timeout 600 python scripts/sweep.py c5host > gpurun_out/r01_c5_host.jsonl 2>&1; echo "c5host exit $?"
