cd $GRAFT_REPO_ROOT
timeout 300 python scripts/py_overhead.py > gpurun_out/r02_py_overhead.jsonl 2>&1; cat gpurun_out/r02_py_overhead.jsonl
