"""Oracle: CFS batch partitioning (A0) and the FCFS baseline.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper, Sec. 7 "Aqua's batch partitioning algorithm":
  "Given a batch size b, we partition it into p prefill tokens and d decode
  tokens. Our key insight to partition is to set d to its upper bound,
  corresponding to the maximum number of prompts that fit within the GPU
  memory. Aqua first fills p with prefill prompts having the least number of
  prefill tokens computed, d with decode prompts with the least number of
  tokens generated. The remaining slots in d are allocated to prompts in p.
  ... Aqua stops filling the batch if the GPU's memory is exhausted."
SPEC's five-step reading: S:265-278.

This follows those steps in order.  Readings:
  R9   ties broken by (arrival, id).
  R10  "remaining slots in d" -> extra prefill tokens for prefill prompts
       already chosen in step 3, in the same order.
  R11  memory test = blocks for current KV + this iteration's tokens:
       need(r, t) = ceil((ctx + t) / bs), summed over included prompts <= NB
       (S:325).
  R12  a prompt that does not fit stops that walk ("stops filling").
  R16  fill order: prefill first, then decode (the paper's sentence order).
  R21  step 4 with no prompt chosen in step 2 (p = 0): the left-over decode
       slots walk the prefill prompts as step 2 does ("empty plan
       only if nothing runnable").
  The count C of step 1 walks prefill-order then decode-order with t = 1
  (each prompt's current KV plus its next token; a prompt with no KV still
  needs one block), stopping at the first that does not fit (R12).
"""
from __future__ import annotations

import dataclasses
from typing import List, Tuple

PREFILL = 0
DECODE = 1


@dataclasses.dataclass
class Req:
    """Per-prompt service counters (D9): prefill tokens computed f, tokens
    generated g, KV tokens stored ctx."""
    id: int
    arrival: float
    P: int            # prompt tokens
    O: int            # output tokens
    f: int = 0
    g: int = 0
    ctx: int = 0
    phase: int = PREFILL


def need(r: Req, t: int, bs: int) -> int:
    """Blocks for r's current KV plus t more tokens (R11)."""
    return -(-(r.ctx + t) // bs)


def decode_order(rs: List[Req]) -> List[Req]:
    """Least tokens generated first; ties (arrival, id) (R9)."""
    return sorted((r for r in rs if r.phase == DECODE), key=lambda r: (r.g, r.arrival, r.id))


def prefill_order(rs: List[Req]) -> List[Req]:
    """Least prefill tokens computed first; ties (arrival, id) (R9)."""
    return sorted((r for r in rs if r.phase == PREFILL), key=lambda r: (r.f, r.arrival, r.id))


def plan(rs: List[Req], b: int, NB: int, bs: int) -> Tuple[List[int], List[Tuple[int, int]]]:
    """partition_batch.  Returns (decode ids,
    [(prefill id, tokens)]), both in selection order.

    The fill order follows the paper's sentence order, "Aqua first fills p
    with prefill prompts ..., d with decode prompts ..." (R16): prefill
    prompts are admitted to memory before decode prompts, which is what
    lets a newly arrived prompt displace the most-served decode prompt
    (fig:cfs_design)."""
    dec = decode_order(rs)
    pre = prefill_order(rs)

    # (1) d = min(b, C): C = number of prompts that fit in memory, walked in
    #     fill order (prefill, then decode) with t = 1 each
    used = 0
    C = 0
    for r in pre + dec:
        n = need(r, 1, bs)
        if used + n > NB:
            break
        used += n
        C += 1
    d = min(b, C)

    # (2) p = b - d prefill tokens, least prefill done first
    used = 0
    p_rem = b - d
    chosen: List[List] = []            # [req, alloc]
    for r in pre:
        if p_rem == 0:
            break
        alloc = min(p_rem, r.P - r.f)
        n = need(r, alloc, bs)
        if used + n > NB:
            break
        used += n
        chosen.append([r, alloc])
        p_rem -= alloc

    # (3) decode prompts, least generated first, while |D| < d and they fit
    D: List[int] = []
    for r in dec:
        if len(D) >= d:
            break
        n = need(r, 1, bs)
        if used + n > NB:
            break
        used += n
        D.append(r.id)

    # (4) leftover decode slots -> extra tokens for the chosen prefill prompts
    left = d - len(D)
    if not chosen and left > 0:
        # R21: step 2 chose no prompt (p = b - d = 0 once >= b prompts fit),
        # so "the remaining slots in d are allocated to prompts in p" means
        # prefill prompts in prefill order, walked as in step 2 with the
        # left-over slots -- otherwise >= b prefill-phase prompts and too few
        # decode prompts would get an empty plan (SPEC partition_batch:
        # "empty plan only if nothing runnable")
        for r in pre:
            if left == 0:
                break
            alloc = min(left, r.P - r.f)
            n = need(r, alloc, bs)
            if used + n > NB:
                break
            used += n
            chosen.append([r, alloc])
            left -= alloc
    for item in chosen:
        if left == 0:
            break
        r, alloc = item
        extra = min(left, r.P - r.f - alloc)
        # (5) the memory test applies here too: shrink until it fits
        while extra > 0 and used - need(r, alloc, bs) + need(r, alloc + extra, bs) > NB:
            extra -= 1
        if extra > 0:
            used += need(r, alloc + extra, bs) - need(r, alloc, bs)
            item[1] = alloc + extra
            left -= extra
    return D, [(r.id, a) for r, a in chosen]


def fcfs_plan(admitted: List[Req], b: int) -> Tuple[List[int], List[Tuple[int, int]]]:
    """Baseline policy (SPEC fcfs_step S:297-305; "admit new
    requests only if there is enough GPU memory"): decode tokens for every
    admitted decode prompt first, the rest of the budget to admitted prefill
    prompts in arrival order (chunked prefill).  Admission itself is done by
    the caller (full KV projection must fit; never preempts)."""
    D = [r.id for r in sorted(admitted, key=lambda r: (r.arrival, r.id)) if r.phase == DECODE][:b]
    rem = b - len(D)
    pre = []
    for r in sorted(admitted, key=lambda r: (r.arrival, r.id)):
        if r.phase != PREFILL or rem == 0:
            continue
        t = min(rem, r.P - r.f)
        pre.append((r.id, t))
        rem -= t
    return D, pre
