cd $GRAFT_REPO_ROOT
timeout 900 python scripts/sweep.py small_chunks2 > gpurun_out/r02_small_chunks2.jsonl 2>gpurun_out/err.log; cut -c1-170 gpurun_out/r02_small_chunks2.jsonl; tail -2 gpurun_out/err.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "ldst_pack" > gpurun_out/r02_pack_tests.log 2>&1; echo "pack tests rc $?"; tail -2 gpurun_out/r02_pack_tests.log
