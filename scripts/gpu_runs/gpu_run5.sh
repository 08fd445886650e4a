cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 2>&1 | tail -4
timeout 400 python bench.py --steps 30 --warmup 5 --cpu-seconds 10 > gpurun_out/r01_bench3.json 2> gpurun_out/r01_bench3.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/r01_bench3.json')); print(d['value'], d['roofline'], d['preempt_resume_ms'], d['e2e']['value'])"
AQUA_BENCH_SHARED_GPU=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r01_bench_n2shared.json 2> gpurun_out/r01_bench_n2shared.err; echo "n2 shared exit $?"; tail -c 600 gpurun_out/r01_bench_n2shared.json; tail -n 5 gpurun_out/r01_bench_n2shared.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/r01_ref_n2.json 2> gpurun_out/r01_ref_n2.err; echo "ref n2 exit $?"; head -c 300 gpurun_out/r01_ref_n2.json
timeout 600 python scripts/c3_run.py --policy cfs-peer --check-oracle > gpurun_out/r01_c3_peer.json 2> gpurun_out/r01_c3_peer.err; echo "c3 peer exit $?"
timeout 900 python scripts/c3_run.py --policy cfs-host > gpurun_out/r01_c3_host.json 2> gpurun_out/r01_c3_host.err; echo "c3 host exit $?"
cat gpurun_out/r01_c3_peer.json gpurun_out/r01_c3_host.json; tail -n 3 gpurun_out/r01_c3_host.err
for t in memcheck racecheck synccheck; do timeout 600 compute-sanitizer --tool $t --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01_sanitizer_$t.log 2>&1; echo "sanitizer $t exit $?"; tail -n 3 gpurun_out/r01_sanitizer_$t.log; done
