"""C3 trace driver: the native CFS scheduler (aqua_cfs) deciding, libaqua
paging, and the synthetic decode writing each iteration's KV (harness for
BASELINE configs[2]; paper Sec. 7 P:836-838 and Sec. 9).

Streams (R7, A8): the swap stream waits for the decode stream before a
swap_out (the blocks' last writer), and the decode stream waits for a
swap_in ticket only before the iteration that needs those prompts -- so
paging overlaps decode instead of the paper's loop-boundary quiescence
(P:866).  With a dry-run ctx (no GPU) only the bookkeeping runs.

The call log has the oracle's format (oracle/sim.py) so the two can be
compared exactly; the driver itself never imports the oracle.
"""
from __future__ import annotations

import time
from typing import Callable, List, Optional, Sequence, Tuple

from . import aqua
from .cfs import Scheduler


def run_trace(trace: Sequence[Tuple[int, float, int, int]], ctx: "aqua.Ctx", sched: Scheduler, *,
              fill_seed: Optional[int] = None, decode_stream: int = 0, swap_stream: int = 0,
              on_iteration: Optional[Callable] = None, record_log: bool = True,
              stream_sync: Optional[Callable] = None, on_swap: Optional[Callable] = None):
    """Run the whole trace.  Returns (log, stats).

    ``stream_sync(kind, ticket)`` lets a GPU caller order streams:
      kind == "before_swap_out": swap stream must wait for decode;
      kind == "before_swap_in":  (timing hook);
      kind == "after_swap_in":   decode must wait for the swap_in ticket.
    ``on_iteration(i, work)`` runs the per-iteration decode proxy (optional).
    ``on_swap(kind, pids, ticket, nblocks)`` is called after each swap call.
    """
    pending = sorted(trace, key=lambda x: (x[1], x[0]))
    pi = 0
    log: List[tuple] = []
    i = 0
    blocks_out = blocks_in = 0
    swap_calls = []
    while True:
        t = sched.vclock()
        while pi < len(pending) and pending[pi][1] <= t:
            rid, a, P, O = pending[pi]
            sched.add(rid, a, P, O)
            pi += 1
        res, outs, ins, work = sched.next()
        if not work:
            if pi >= len(pending):
                break
            sched.advance_to(pending[pi][1])
            continue
        if res and record_log:
            D, PF = sched.partition()
            log.append(("plan", i, tuple(D), tuple((p, t) for p, t in PF)))
        if outs:
            if stream_sync:
                stream_sync("before_swap_out", 0)
            t0 = time.perf_counter()
            tk = ctx.swap_out(outs, swap_stream)
            q = [ctx.query(p, with_ids=True) for p in outs]
            n = sum(x[2] for x in q)
            blocks_out += n
            swap_calls.append(("out", n, tk, t0))
            if on_swap:
                on_swap("out", outs, tk, n)
            if record_log:
                log.append(("swap_out", tuple(outs), tuple((x[1], tuple(x[3])) for x in q)))
        if ins:
            if stream_sync:
                stream_sync("before_swap_in", 0)
            t0 = time.perf_counter()
            new, tk = ctx.swap_in(ins, swap_stream)
            n = sum(len(x) for x in new)
            blocks_in += n
            swap_calls.append(("in", n, tk, t0))
            if stream_sync:
                stream_sync("after_swap_in", tk)
            if on_swap:
                on_swap("in", ins, tk, n)
            if record_log:
                log.append(("swap_in", tuple(ins), tuple(tuple(x) for x in new)))
        for pid, ctx0, tok, grow, phase in work:
            if grow > 0:
                ids = ctx.alloc_blocks(pid, grow, decode_stream)
                if record_log:
                    log.append(("alloc", pid, tuple(ids)))
        if record_log:
            log.append(("iter", i, tuple((pid, ctx0, tok) for pid, ctx0, tok, _, _ in work)))
        if fill_seed is not None:
            for pid, ctx0, tok, _, _ in work:
                ctx.kv_fill_pattern(pid, ctx0, ctx0 + tok, fill_seed, decode_stream)
        if on_iteration:
            on_iteration(i, work)
        fin, _ = sched.commit()
        for pid in fin:
            ctx.free(pid, decode_stream)
            if record_log:
                log.append(("free", pid))
        i += 1
    return log, {"iters": i, "blocks_out": blocks_out, "blocks_in": blocks_in, "swap_calls": swap_calls,
                 "vclock": sched.vclock()}
