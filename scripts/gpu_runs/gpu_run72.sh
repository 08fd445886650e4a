cd $GRAFT_REPO_ROOT
for pk in 0 64 128; do
AQUA_LDST_PACK=$pk timeout 900 python scripts/sweep.py small_chunks > gpurun_out/r01_small_chunks_pack$pk.jsonl 2>gpurun_out/err.log
echo "pack $pk"; grep '"variant": 3, "sched": 2\|"sched": "auto"' gpurun_out/r01_small_chunks_pack$pk.jsonl | grep -v '"S": 4096\|"S": 8192' | cut -c1-150
done
