"""Seeded synthetic inputs.

Seeds: KV content 0, block permutation 2, trace 1 unless a test says
otherwise.  KV values are uniform random 16-bit words over the full range
(NaN / Inf / subnormal bf16 patterns included) so that any accidental
floating-point path breaks bit-exactness.
"""
from __future__ import annotations

import dataclasses
from typing import List, Tuple

import numpy as np


@dataclasses.dataclass(frozen=True)
class KVShape:
    name: str
    L: int       # layers
    H: int       # KV heads (per TP shard)
    D: int       # head dim
    e: int       # element bytes (2: fp16 / bf16)
    bs: int      # tokens per block

    @property
    def S(self) -> int:
        return self.bs * self.H * self.D * self.e

    @property
    def U(self) -> int:
        return 2 * self.L * self.S


# BASELINE.json configs (shapes only; the workloads are described in DESIGN.md)
CONFIGS = {
    "tiny": KVShape("tiny", L=2, H=2, D=64, e=2, bs=16),                 # configs[0]
    "llama3-8b": KVShape("llama3-8b", L=32, H=8, D=128, e=2, bs=16),     # configs[1], [2], [4]
    "llama3-70b-tp4": KVShape("llama3-70b-tp4", L=80, H=2, D=128, e=2, bs=16),  # configs[3]
}


def kv_random_bytes(nbytes: int, seed: int = 0) -> np.ndarray:
    """uint8[nbytes] of uniform random 16-bit words (little-endian)."""
    assert nbytes % 2 == 0
    w = np.random.default_rng(seed).integers(0, 1 << 16, size=nbytes // 2, dtype=np.uint16)
    return w.view(np.uint8)


def block_permutation(nb: int, n: int, seed: int = 2) -> np.ndarray:
    """The first n ids of a seeded permutation of range(nb): a fragmented,
    non-monotone block table (worst case for the gather)."""
    return np.random.default_rng(seed).permutation(nb)[:n].astype(np.int32)


def lognormal_lengths(rng: np.random.Generator, n: int, median: float, sigma: float,
                      lo: int, hi: int) -> np.ndarray:
    """Lognormal(log(median), sigma) rounded to int, truncated to [lo, hi] by
    resampling ("sharegpt-like")."""
    out = np.empty(n, dtype=np.int64)
    filled = 0
    while filled < n:
        x = np.rint(rng.lognormal(np.log(median), sigma, size=n)).astype(np.int64)
        x = x[(x >= lo) & (x <= hi)]
        take = min(n - filled, x.size)
        out[filled:filled + take] = x[:take]
        filled += take
    return out


def burst_trace(seed: int = 1, lam0: float = 2.5, n_pre: int = 25, burst_mult: float = 2.0,
                burst_s: float = 60.0, tail_s: float = 15.0,
                prompt=(2000, 0.8, 1, 8192), output=(250, 0.7, 1, 2048)) -> List[Tuple[int, float, int, int]]:
    """BASELINE configs[2]: 25 prompts at lam0, then burst_mult*lam0 for
    burst_s seconds ("25 prompts ... double the request rate for one
    minute"), then lam0 for tail_s seconds; Poisson arrivals; sharegpt-like
    truncated-lognormal lengths.  Returns [(id, arrival_s, P, O)]."""
    rng = np.random.default_rng(seed)
    arr: List[float] = []
    t = 0.0
    for _ in range(n_pre):
        t += rng.exponential(1.0 / lam0)
        arr.append(t)
    t0 = t
    for rate, end in ((lam0 * burst_mult, t0 + burst_s), (lam0, t0 + burst_s + tail_s)):
        while True:
            t += rng.exponential(1.0 / rate)
            if t >= end:
                t = end
                break
            arr.append(t)
    n = len(arr)
    P = lognormal_lengths(rng, n, *prompt)
    O = lognormal_lengths(rng, n, *output)
    return [(i, float(arr[i]), int(P[i]), int(O[i])) for i in range(n)]
