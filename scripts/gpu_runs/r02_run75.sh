cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider > gpurun_out/r02_parity_split.log 2>&1; echo "parity rc $?"; tail -3 gpurun_out/r02_parity_split.log
timeout 600 python scripts/overlap.py --images mixed,mixed_tma --decode gemm --reps 3 > gpurun_out/r02_mixed_split.jsonl 2> gpurun_out/r02_mixed_split.err; echo "overlap gemm rc $?"
timeout 600 python scripts/overlap.py --images mixed,mixed_tma --decode hbm --reps 3 >> gpurun_out/r02_mixed_split.jsonl 2>> gpurun_out/r02_mixed_split.err; echo "overlap hbm rc $?"
cat gpurun_out/r02_mixed_split.jsonl; tail -3 gpurun_out/r02_mixed_split.err
