cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -4
timeout 600 python scripts/sweep.py prefix > gpurun_out/r01_prefix.jsonl 2>&1; echo "prefix $?"; cat gpurun_out/r01_prefix.jsonl
B="python bench.py --steps 3 --warmup 3 --no-host-baselines --no-cpu-baseline"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv $B > /dev/null 2>&1; echo "launch list $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:swap_tma_kernel -s 6 -c 2 -o gpurun_out/r01_prof_tma_final $B > gpurun_out/ncu_full2.log 2>&1; echo "full $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:swap_tma_kernel -s 6 -c 2 -o gpurun_out/r01_prof_tma_c4 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full3.log 2>&1; echo "full c4 $?"
