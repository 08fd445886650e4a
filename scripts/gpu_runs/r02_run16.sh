cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/r02_bench_final.json 2> gpurun_out/r02_bench_final.err; echo "bench rc $?"; head -c 400 gpurun_out/r02_bench_final.json; echo
timeout 900 python bench.py --config c4 --no-host-baselines > gpurun_out/r02_bench_c4_final.json 2> gpurun_out/r02_bench_c4_final.err; echo "bench c4 rc $?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_bench_reference.json 2>&1; echo "ref rc $?"; cat gpurun_out/r02_bench_reference.json | head -c 300; echo
timeout 900 python scripts/c3_run.py --policy cfs-peer --check-oracle > gpurun_out/r02_c3_peer.json 2> gpurun_out/r02_c3.err; echo "c3 rc $?"; head -c 600 gpurun_out/r02_c3_peer.json; echo
timeout 900 python scripts/c3_run.py --policy cfs-host --exchange --check-oracle > gpurun_out/r02_c3_host_exchange.json 2>> gpurun_out/r02_c3.err; echo "c3 host rc $?"; head -c 600 gpurun_out/r02_c3_host_exchange.json; echo
tail -3 gpurun_out/r02_c3.err
