cd $GRAFT_REPO_ROOT
AQUA_SWEEP_S=512 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:swap_small -s 4 -c 1 -o gpurun_out/r02_prof_small512 python scripts/sweep.py small_ldst > gpurun_out/r02_prof_small512.log 2>&1; echo "rc $?"; tail -3 gpurun_out/r02_prof_small512.log
