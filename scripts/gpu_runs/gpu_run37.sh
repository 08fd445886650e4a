cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf --timeout 300 -k "tma_r4 or tma_ws" 2>&1 | tail -5
AQUA_SWEEP_TMA_VARIANTS=0,2,3 AQUA_SWEEP_STAGES=0,3,4,6 timeout 400 python scripts/sweep.py tma_variants > gpurun_out/r01_tma_rings.jsonl 2>&1; cat gpurun_out/r01_tma_rings.jsonl
