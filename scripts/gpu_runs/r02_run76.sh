cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke_split.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/r02_smoke_split.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_gpu_suite_split.log 2>&1; echo "gpu suite rc $?"; tail -2 gpurun_out/r02_gpu_suite_split.log
SEL="mixed_arena or degenerate_and_maximum or host_engines_switching or copy_engine_staging"
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --leak-check full --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "$SEL" -p no:cacheprovider > gpurun_out/r02_memcheck_split.log 2>&1; echo "memcheck rc $?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/r02_memcheck_split.log | tail -3
