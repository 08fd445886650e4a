cd $GRAFT_REPO_ROOT
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 400 python bench.py > gpurun_out/r01_bench_end2.json 2> gpurun_out/bench.err; echo "bench exit $?"
python -c "import json;d=json.load(open('gpurun_out/r01_bench_end2.json'));print(d['value'], d['roofline']['achieved'], d['roofline']['swap_in_achieved'], d['roofline']['rw_bound']['frac'], d['e2e']['value'], d['clocks'])"
timeout 300 python bench.py --config c4 --no-host-baselines --no-cpu-baseline > gpurun_out/r01_bench_c4_end2.json 2>>gpurun_out/bench.err; python -c "import json;d=json.load(open('gpurun_out/r01_bench_c4_end2.json'));print('c4', d['value'], d['roofline']['achieved'], d['parity'])"
B="python bench.py --steps 3 --warmup 3 --no-host-baselines --no-cpu-baseline"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_end.csv $B > /dev/null 2>&1; echo "launch list $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:swap_tma_kernel -s 6 -c 2 -o gpurun_out/r01_prof_tma_end $B > gpurun_out/ncu_end.log 2>&1; echo "full $?"
