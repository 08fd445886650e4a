cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r02_gpu_suite2.log 2>&1; echo "suite rc $?"; tail -3 gpurun_out/r02_gpu_suite2.log
timeout 900 python scripts/sweep.py small_chunks > gpurun_out/r02_small_chunks_ww.jsonl 2>gpurun_out/err.log; cut -c1-150 gpurun_out/r02_small_chunks_ww.jsonl; tail -2 gpurun_out/err.log
timeout 600 python bench.py --no-host-baselines --no-cpu-baseline > gpurun_out/r02_bench2.json 2> gpurun_out/r02_bench2.err; echo "bench rc $?"; python -c "
import json;d=json.load(open('gpurun_out/r02_bench2.json'));print(d['value'], d['roofline']['achieved'], d['roofline']['swap_in_achieved'], d['e2e']['value'], d['launch_shape'])"
timeout 600 python bench.py --config c4 --no-host-baselines --no-cpu-baseline > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err; python -c "
import json;d=json.load(open('gpurun_out/r02_bench_c4.json'));print(d['value'], d['roofline']['achieved'], d['roofline']['swap_in_achieved'])"
