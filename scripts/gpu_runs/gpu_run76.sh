cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 300 -x 2>&1 | tail -3
timeout 400 python bench.py --no-host-baselines --no-cpu-baseline > gpurun_out/b76.json 2>gpurun_out/bench.err; python -c "import json;d=json.load(open('gpurun_out/b76.json'));print(d['value'], d['roofline']['achieved'], d['launch_shape']['schedule'])"
