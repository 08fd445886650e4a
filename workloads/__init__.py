"""Seeded synthetic inputs shared by the tests, bench.py and the oracle.

Holds NONE of the method's arithmetic: only random bytes, permutations and
request traces.  Both the oracle and the CUDA path
consume these inputs; neither side's results are ever produced here.
"""
from .gen import (CONFIGS, KVShape, burst_trace, kv_random_bytes, block_permutation,
                  lognormal_lengths)

__all__ = ["CONFIGS", "KVShape", "burst_trace", "kv_random_bytes", "block_permutation",
           "lognormal_lengths"]
