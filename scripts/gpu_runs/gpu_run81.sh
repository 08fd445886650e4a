cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 300 -x 2>&1 | tail -2
timeout 400 python scripts/sweep.py engines > gpurun_out/r01_engines_end2.jsonl 2> gpurun_out/err.log; grep '"max_ctas": 0' gpurun_out/r01_engines_end2.jsonl | cut -c1-200
