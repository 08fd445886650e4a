cd $GRAFT_REPO_ROOT
timeout 900 python scripts/overlap.py --decode gemm --images self,host --caps 0,64,32,16,8 --steps 8 > gpurun_out/r02_overlap_gemm.jsonl 2>gpurun_out/err.log; echo "rc $?"; cat gpurun_out/r02_overlap_gemm.jsonl; tail -3 gpurun_out/err.log
