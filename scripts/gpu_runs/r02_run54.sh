cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke_s3.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/r02_smoke_s3.log
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_gpu_suite_s3.log 2>&1; echo "gpu suite rc $?"; tail -3 gpurun_out/r02_gpu_suite_s3.log
timeout 600 python bench.py > gpurun_out/r02_bench_s3.json 2> gpurun_out/r02_bench_s3.err; echo "bench rc $?"; cat gpurun_out/r02_bench_s3.json | head -c 600; echo
timeout 600 python bench.py --config c4 > gpurun_out/r02_bench_c4_s3.json 2>> gpurun_out/r02_bench_s3.err; echo "bench c4 rc $?"
timeout 600 python bench.py --impl reference > gpurun_out/r02_bench_ref_s3.json 2>> gpurun_out/r02_bench_s3.err; echo "ref rc $?"; head -c 400 gpurun_out/r02_bench_ref_s3.json; echo
tail -3 gpurun_out/r02_bench_s3.err
