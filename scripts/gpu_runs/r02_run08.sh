cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r02_gpu_suite3.log 2>&1; echo "suite rc $?"; tail -3 gpurun_out/r02_gpu_suite3.log
AQUA_SWEEP_S=512,1024,2048,4096,8192,32768 timeout 900 python scripts/sweep.py small_chunks2 > gpurun_out/r02_small_chunks_final.jsonl 2>gpurun_out/err.log; grep auto gpurun_out/r02_small_chunks_final.jsonl | cut -c1-200; tail -2 gpurun_out/err.log
timeout 600 python bench.py --no-host-baselines --no-cpu-baseline > gpurun_out/r02_bench3.json 2> gpurun_out/r02_bench3.err; echo "bench rc $?"; python -c "
import json;d=json.load(open('gpurun_out/r02_bench3.json'));print(d['value'], d['roofline']['achieved'], d['roofline']['swap_in_achieved'], d['e2e']['value'])"
timeout 600 python bench.py --config c4 --no-host-baselines --no-cpu-baseline > gpurun_out/r02_bench_c4b.json 2> gpurun_out/r02_bench_c4b.err; python -c "
import json;d=json.load(open('gpurun_out/r02_bench_c4b.json'));print(d['value'], d['roofline']['achieved'], d['roofline']['swap_in_achieved'], d['launch_shape'])"
