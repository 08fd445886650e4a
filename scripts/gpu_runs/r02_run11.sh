cd $GRAFT_REPO_ROOT
timeout 900 python scripts/overlap.py > gpurun_out/r02_overlap.jsonl 2> gpurun_out/r02_overlap.err; echo "overlap rc $?"; cat gpurun_out/r02_overlap.jsonl; tail -2 gpurun_out/r02_overlap.err
# launch list of the bench command (cold-cache, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-host-baselines --no-cpu-baseline > gpurun_out/r02_launches_bench.log 2>&1; echo "launches rc $?"
# full capture of the product kernel: C2 swap_out / swap_in (after warm-up), C4, and the 1 KiB / 512 B small-chunk shapes
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:swap_tma -s 8 -c 2 -o gpurun_out/r02_prof_c2 python bench.py --steps 2 --warmup 3 --no-host-baselines --no-cpu-baseline > gpurun_out/r02_prof_c2.log 2>&1; echo "prof c2 rc $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:swap_tma -s 8 -c 2 -o gpurun_out/r02_prof_c4 python bench.py --config c4 --steps 2 --warmup 3 --no-host-baselines --no-cpu-baseline > gpurun_out/r02_prof_c4.log 2>&1; echo "prof c4 rc $?"
AQUA_SWEEP_S=1024,512 AQUA_SWEEP_ENGINES=auto timeout 1200 ncu --set full --clock-control none --import-source on -k regex:swap_tma -s 10 -c 2 -o gpurun_out/r02_prof_small python scripts/sweep.py small_chunks2 > gpurun_out/r02_prof_small.log 2>&1; echo "prof small rc $?"
ls -la gpurun_out/*.ncu-rep
