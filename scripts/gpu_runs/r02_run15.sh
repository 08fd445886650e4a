cd $GRAFT_REPO_ROOT
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="test_c1_bytes or (test_random_sequences_bytes and (s512 or s1k or s2k or c4_shape or tiny_256B or llama_bs32)) or test_multistream_fuzz or test_swap_exchange_bytes or test_block_major or host_engines or host_staging"
timeout 1500 $CS --tool memcheck --leak-check full --print-limit 100000 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py -q -m gpu -k "$SEL or peer_policy" -p no:cacheprovider > gpurun_out/r02_sanitizer_memcheck.log 2>&1; echo "memcheck rc $?"; grep -E "ERROR SUMMARY|LEAK SUMMARY|passed|failed" gpurun_out/r02_sanitizer_memcheck.log | tail -4
python - <<'PY'
import re, collections
txt=open('gpurun_out/r02_sanitizer_memcheck.log').read()
blocks=txt.split('========= Leaked ')[1:]
c=collections.Counter('libaqua' if 'libaqua' in b[:400] else 'torch/cudart' for b in blocks)
print("leaked allocations by owner:", dict(c))
PY
