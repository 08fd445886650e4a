cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "hybrid or auto_policy or dyn" > gpurun_out/r02_claims_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/r02_claims_tests.log
for lu in 0 1 2 4; do
AQUA_HYBRID_LDST_UNITS=$lu AQUA_SWEEP_S=512,1024,2048 AQUA_SWEEP_ENGINES=hybrid,ring AQUA_SWEEP_HYBRID_UNITS=2,4,8,16,32 timeout 900 python scripts/sweep.py small_chunks2 >> gpurun_out/r02_hybrid_split.jsonl 2>>gpurun_out/err.log
done
tail -2 gpurun_out/err.log
