cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py -q -m gpu -p no:cacheprovider > gpurun_out/r02_parity_split2.log 2>&1; echo "parity rc $?"; tail -3 gpurun_out/r02_parity_split2.log
timeout 2400 python scripts/product_mutants.py run --kind gpu --only "AUTO: a call with images in both,AUTO: the split sends,AUTO: layer-wise mixed" --timeout 600 --out gpurun_out/r02_product_mutants_gpu_split.json > gpurun_out/r02_product_mutants_gpu_split.log 2>&1; echo "mutants rc $?"; tail -8 gpurun_out/r02_product_mutants_gpu_split.log
