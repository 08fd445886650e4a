"""Oracle: closed-form synthetic KV content (C-11).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Not a paper formula: a test-design device so that the KV bytes a prompt
must hold are known at any time without replaying its swap history (the
restore invariant "KV bytes ... conserved across swaps", made
checkable at full scale).  The GPU side implements the same counter-based
generator independently (paper_2407_21255_b200/csrc); nothing is shared.

  word(p, t, l, kv, h, d) = low 16 bits of splitmix64(seed XOR pack)
  pack = p<<46 | t<<26 | l<<18 | kv<<17 | h<<10 | d
  splitmix64(x): z = x + 0x9E3779B97F4A7C15
                 z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
                 z = (z ^ (z >> 27)) * 0x94D049BB133111EB
                 return z ^ (z >> 31)            (all mod 2**64)

Token t of prompt p lives in block bt[t // bs], row i = t % bs; element
(h, d) of that token is the little-endian 16-bit word at element offset
(i*H + h)*D + d of chunk (l, kv) (flash layout [bs][H][D], e = 2).
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1


def splitmix64_int(x: int) -> int:
    """Scalar reference, Python integers mod 2**64."""
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised over uint64 arrays (NumPy uint64 arithmetic wraps mod 2**64)."""
    x = x.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def pack(p, t, l, kv, h, d):
    u = np.uint64
    return ((u(p) << u(46)) | (np.asarray(t, dtype=np.uint64) << u(26)) | (u(l) << u(18))
            | (u(kv) << u(17)) | (np.asarray(h, dtype=np.uint64) << u(10)) | np.asarray(d, dtype=np.uint64))


def token_words(seed: int, p: int, t: int, l: int, kv: int, H: int, D: int) -> np.ndarray:
    """uint16[H, D]: the words of token t of prompt p at (layer l, kv)."""
    h = np.arange(H, dtype=np.uint64)[:, None]
    d = np.arange(D, dtype=np.uint64)[None, :]
    z = splitmix64(np.uint64(seed) ^ pack(p, np.uint64(t), l, kv, h, d))
    return (z & np.uint64(0xFFFF)).astype(np.uint16)


def write_tokens(pool, pid: int, t0: int, t1: int, seed: int) -> None:
    """Synthetic decode/prefill: store tokens [t0, t1) of pid into its blocks
    (bytes-mode kvpool.Pool, e = 2)."""
    lay = pool.lay
    assert lay.e == 2
    bt = pool.prompts[pid].blocks
    for t in range(t0, t1):
        b, i = bt[t // lay.bs], t % lay.bs
        for l in range(lay.L):
            for kv in (0, 1):
                w = token_words(seed, pid, t, l, kv, lay.H, lay.D)
                ch = pool.chunk(l, kv, b)
                row = i * lay.H * lay.D * 2
                ch[row:row + lay.H * lay.D * 2] = w.reshape(-1).view(np.uint8)


def write_token_range(pool, pid: int, t0: int, t1: int, seed: int) -> None:
    """write_tokens for a whole range at once (same bytes): the words of
    tokens [t0, t1) are computed together per (layer, kv), then stored one
    run of consecutive rows per block."""
    lay = pool.lay
    assert lay.e == 2
    if t1 <= t0:
        return
    bt = pool.prompts[pid].blocks
    row = lay.H * lay.D * 2
    t = np.arange(t0, t1, dtype=np.uint64)[:, None, None]
    h = np.arange(lay.H, dtype=np.uint64)[None, :, None]
    d = np.arange(lay.D, dtype=np.uint64)[None, None, :]
    for l in range(lay.L):
        for kv in (0, 1):
            z = splitmix64(np.uint64(seed) ^ pack(pid, t, l, kv, h, d))
            w = (z & np.uint64(0xFFFF)).astype(np.uint16).reshape(t1 - t0, row // 2).view(np.uint8)
            tt = t0
            while tt < t1:
                b, i = bt[tt // lay.bs], tt % lay.bs
                n = min(lay.bs - i, t1 - tt)
                ch = pool.chunk(l, kv, b)
                ch[i * row:(i + n) * row] = w[tt - t0:tt - t0 + n].reshape(-1)
                tt += n


def check_tokens(pool, pid: int, ntok: int, seed: int) -> bool:
    """True iff tokens [0, ntok) of pid hold their closed-form words."""
    lay = pool.lay
    bt = pool.prompts[pid].blocks
    for t in range(ntok):
        b, i = bt[t // lay.bs], t % lay.bs
        for l in range(lay.L):
            for kv in (0, 1):
                w = token_words(seed, pid, t, l, kv, lay.H, lay.D)
                ch = pool.chunk(l, kv, b)
                row = i * lay.H * lay.D * 2
                if not np.array_equal(ch[row:row + lay.H * lay.D * 2], w.reshape(-1).view(np.uint8)):
                    return False
    return True
