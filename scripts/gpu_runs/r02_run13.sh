cd $GRAFT_REPO_ROOT
for tu in 0 1 2 4; do for tm in 1 2 4; do
if [ $tu = 0 ] && [ $tm != 2 ]; then continue; fi
AQUA_TAIL_UNITS=$tu AQUA_TAIL_MULT=$tm AQUA_SWEEP_S=512,1024,2048 AQUA_SWEEP_ENGINES=auto timeout 900 python scripts/sweep.py small_chunks2 | sed "s/^{/{\"tail_units\": $tu, \"tail_mult\": $tm, /" >> gpurun_out/r02_tail.jsonl 2>>gpurun_out/err.log
done; done
tail -2 gpurun_out/err.log
