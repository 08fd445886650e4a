cd $GRAFT_REPO_ROOT
CS=/usr/local/cuda/bin/compute-sanitizer
for e in tma ldst; do timeout 300 $CS --tool initcheck --print-limit 3 python scripts/initcheck_probe.py $e > gpurun_out/r02_initcheck_probe_$e.log 2>&1; echo "$e rc $?"; grep -E "arena bytes|ERROR SUMMARY|Uninitialized" gpurun_out/r02_initcheck_probe_$e.log | head -4; done
