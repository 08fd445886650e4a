cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf --timeout 300 -k "tma_ws" 2>&1 | tail -5
timeout 300 python scripts/sweep.py tma_variants > gpurun_out/r01_tma_variants.jsonl 2>&1; tail -40 gpurun_out/r01_tma_variants.jsonl
