"""B200-native preempt/resume KV paging (arXiv 2407.21255, "Aqua").

The product is the C-ABI library ``libaqua.so`` (include/aqua.h, sources in
csrc/) and its thin ctypes binding ``paper_2407_21255_b200.aqua``.  Importing
``.aqua`` fails loudly if the library has not been built; there is no CPU
fallback.  Build with ``python -m paper_2407_21255_b200.build``.
"""
