cd $GRAFT_REPO_ROOT
timeout 900 python scripts/overlap.py --images host,self,mixed,mixed_tma --decode hbm > gpurun_out/r02_overlap_final.jsonl 2> gpurun_out/r02_overlap_final.err; echo "hbm rc $?"
timeout 900 python scripts/overlap.py --images host,mixed,mixed_tma,self --caps 0,32 --decode gemm >> gpurun_out/r02_overlap_final.jsonl 2>> gpurun_out/r02_overlap_final.err; echo "gemm rc $?"
cat gpurun_out/r02_overlap_final.jsonl; tail -2 gpurun_out/r02_overlap_final.err
