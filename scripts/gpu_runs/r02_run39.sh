cd $GRAFT_REPO_ROOT
for S in 512 1024; do
AQUA_SWEEP_S=$S timeout 900 ncu --set full --clock-control none --import-source on -k regex:swap_small -s 4 -c 2 -o gpurun_out/r02_prof_small_auto$S python scripts/sweep.py ncu_small > gpurun_out/r02_prof_small_auto$S.log 2>&1; echo "rc $?"; tail -2 gpurun_out/r02_prof_small_auto$S.log
done
