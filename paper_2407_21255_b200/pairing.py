"""Borrower -> lender pairing and the one setup-time exchange of IPC handles
(paper Sec. 5: one producer per consumer).

On an NVSwitch box every GPU pair has the same bandwidth, so the lowest-index
perfect matching r <-> r^1 is used (an odd last rank lends to itself).  The
only cross-process traffic is this exchange of 64-byte handles through
torch.distributed; the data path has no collective.
"""
from __future__ import annotations

from typing import List, Optional, Sequence


def partner(rank: int, world: int, can_access: Optional[Sequence[Sequence[bool]]] = None) -> int:
    """Lender of `rank`.  With a P2P reachability matrix, pairs that cannot
    reach each other fall back to self-lending."""
    p = rank ^ 1
    if p >= world:
        return rank
    if can_access is not None and not (can_access[rank][p] and can_access[p][rank]):
        return rank
    return p


def best_matching(bw: Sequence[Sequence[float]]) -> List[int]:
    """Lender of every GPU from a measured P2P bandwidth matrix bw[i][j]
    (GB/s; 0 = unreachable): the perfect matching (odd count: one GPU lends
    to itself) that maximises the minimum of min(bw[i][j], bw[j][i]) over
    its pairs; ties -> lexicographically smallest partner list.  Brute force
    over all matchings (105 for 8 GPUs)."""
    n = len(bw)
    best, best_key = None, None

    def rec(free, part):
        nonlocal best, best_key
        if not free:
            vals = [min(bw[i][part[i]], bw[part[i]][i]) for i in range(n) if part[i] != i]
            key = (min(vals) if vals else float("inf"), [-x for x in part])
            if best_key is None or key > best_key:
                best, best_key = list(part), key
            return
        i = free[0]
        rest = free[1:]
        if len(free) % 2 == 1:          # odd: i may lend to itself
            part[i] = i
            rec(rest, part)
        for k, j in enumerate(rest):
            part[i], part[j] = j, i
            rec(rest[:k] + rest[k + 1:], part)
        part[i] = -1

    rec(list(range(n)), [-1] * n)
    return best


def best_bipartite(bw: Sequence[Sequence[float]], borrowers: Sequence[int], lenders: Sequence[int]) -> List[int]:
    """Split roles (BASELINE configs[3]: borrower GPUs each paging to one of
    as many lender GPUs): the one-to-one assignment of lenders to
    borrowers that maximises the minimum link bandwidth min(bw[b][l],
    bw[l][b]) over its pairs; ties -> lexicographically smallest partner
    list.  Returns partner[r] for every rank (a borrower's lender, a
    lender's borrower; ranks in neither list map to themselves).  Brute
    force over permutations (24 for 4 + 4 GPUs)."""
    import itertools
    if len(borrowers) != len(lenders):
        raise ValueError("split roles need as many lenders as borrowers")
    n = len(bw)
    best, best_key = None, None
    for perm in itertools.permutations(lenders):
        part = list(range(n))
        for b, l in zip(borrowers, perm):
            part[b], part[l] = l, b
        vals = [min(bw[b][l], bw[l][b]) for b, l in zip(borrowers, perm)]
        key = (min(vals) if vals else float("inf"), [-x for x in part])
        if best_key is None or key > best_key:
            best, best_key = part, key
    return best


def measure_p2p(ndev: int, nbytes: int = 256 << 20, reps: int = 3) -> List[List[float]]:
    """Measured device-to-device copy bandwidth (GB/s) between every pair of
    the visible GPUs (one process, torch copies; setup only).  0 where P2P
    is not possible."""
    import torch
    from . import aqua
    bufs = [torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{d}") for d in range(ndev)]
    bw = [[0.0] * ndev for _ in range(ndev)]
    for i in range(ndev):
        for j in range(ndev):
            if i == j or not aqua.can_access_peer(i, j):
                continue
            torch.cuda.set_device(i)
            bufs[j].copy_(bufs[i])
            torch.cuda.synchronize(i)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                bufs[j].copy_(bufs[i])
            b.record()
            torch.cuda.synchronize(i)
            torch.cuda.synchronize(j)
            bw[i][j] = reps * nbytes / (a.elapsed_time(b) / 1e3) / 1e9
    return bw


def exchange(obj, group=None) -> List:
    """all_gather_object of a small picklable object (the IPC handle and
    its size) -- setup only."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out
