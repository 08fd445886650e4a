cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -3
timeout 400 python bench.py > gpurun_out/r01_bench_end.json 2> gpurun_out/bench.err; echo "bench exit $?"
python -c "import json;d=json.load(open('gpurun_out/r01_bench_end.json'));print(d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['roofline']['rw_bound'], d['e2e']['value'], d['preempt_resume_ms']['sum_device_ms'], d['preempt_resume_vs_host'], d['launch_shape'], d['clocks'], d['cpu_baseline']['value'])"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01_bench_ref_end.json 2>>gpurun_out/bench.err; echo "ref exit $?"; head -c 200 gpurun_out/r01_bench_ref_end.json; echo
timeout 300 python bench.py --config c4 --no-host-baselines --no-cpu-baseline > gpurun_out/r01_bench_c4_end.json 2>>gpurun_out/bench.err; python -c "import json;d=json.load(open('gpurun_out/r01_bench_c4_end.json'));print('c4', d['value'], d['roofline']['achieved'], d['roofline']['traffic'], d['parity'])"
timeout 600 python scripts/c3_run.py --policy cfs-peer --native --exchange --check-oracle > gpurun_out/r01_c3_native_end.json 2> gpurun_out/c3.err; echo "c3 native $?"; python -c "import json;d=json.load(open('gpurun_out/r01_c3_native_end.json'));print(d.get('swap_GBps'), d.get('verify_mismatches'), d.get('oracle_log_equal'), d.get('wall_s'))"; tail -2 gpurun_out/c3.err
AQUA_BENCH_SHARED_GPU=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r01_bench_n2_end.json 2> gpurun_out/n2.err; echo "n2 exit $?"; python -c "import json;d=json.load(open('gpurun_out/r01_bench_n2_end.json'));print('n2', d['value'], d['mode'], d['pairing'], d['parity'])"
