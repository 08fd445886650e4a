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


def exchange(obj, group=None) -> List:
    """all_gather_object of a small picklable object (the IPC handle and
    its size) -- setup only."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out
