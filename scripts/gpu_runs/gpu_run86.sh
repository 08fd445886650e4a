cd $GRAFT_REPO_ROOT
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 400 python bench.py > gpurun_out/b86.json 2> gpurun_out/bench.err; echo "bench exit $?"
python -c "import json;d=json.load(open('gpurun_out/b86.json'));print(d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['e2e']['value'], d['launch_shape']['schedule'], d['parity'])"
