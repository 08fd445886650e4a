cd $GRAFT_REPO_ROOT
for kb in 32 64 256; do
AQUA_PACK_BATCH_KIB=$kb timeout 900 python scripts/sweep.py pack_sweep >> gpurun_out/r02_pack_sweep.jsonl 2>>gpurun_out/err.log
done
cat gpurun_out/r02_pack_sweep.jsonl; tail -2 gpurun_out/err.log
