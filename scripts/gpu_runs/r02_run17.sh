cd $GRAFT_REPO_ROOT
for hw in 4 8 16; do
AQUA_HYBRID_WARPS=$hw AQUA_SWEEP_S=512,1024,2048 AQUA_SWEEP_ENGINES=auto AQUA_SWEEP_HYBRID_UNITS=4,8,16,32 timeout 900 python scripts/sweep.py small_chunks2 | sed "s/^{/{\"hybrid_warps\": $hw, /" >> gpurun_out/r02_hybrid_warps.jsonl 2>>gpurun_out/err.log
for lu in 1 2 4; do
AQUA_HYBRID_WARPS=$hw AQUA_HYBRID_LDST_UNITS=$lu AQUA_SWEEP_S=512,1024 AQUA_SWEEP_ENGINES=none AQUA_SWEEP_HYBRID_UNITS=16,32 timeout 900 python scripts/sweep.py small_chunks2 | sed "s/^{/{\"hybrid_warps\": $hw, /" >> gpurun_out/r02_hybrid_warps.jsonl 2>>gpurun_out/err.log
done; done
tail -2 gpurun_out/err.log
