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
              stream_sync: Optional[Callable] = None, on_swap: Optional[Callable] = None,
              elastic: Optional[dict] = None, policy_after_relend: int = 0,
              exchange_stream: Optional[int] = None, exchange_pieces: int = 16,
              warm: Sequence[int] = (), max_iters: Optional[int] = None):
    """Run the whole trace.  Returns (log, stats).

    ``stream_sync(kind, ticket)`` lets a GPU caller order streams:
      kind == "before_swap_out": swap stream must wait for decode;
      kind == "before_swap_in":  (timing hook);
      kind == "after_swap_in":   decode must wait for the swap_in ticket.
    ``on_iteration(i, work)`` runs the per-iteration decode proxy (optional).
    ``on_swap(kind, pids, ticket, nblocks)`` is called after each swap call.
    ``elastic = {"t_reclaim": s, "t_relend": s, "relend": (device, base, bytes)}``
    ``exchange_stream`` (a second swap stream): a reschedule with both lists
    uses aqua_swap_exchange -- the preemption on swap_stream, the resume on
    exchange_stream, pipelined in exchange_pieces -- so both link directions
    are busy together (same ids, slots and bytes as the two calls).
    replays NEXT-1: at the first iteration at or after t_reclaim the lender
    takes its memory back (aqua_reclaim: images move to host DRAM) and the
    scheduler falls back to FCFS; at t_relend the memory is
    offered again, the host images move back (ascending pid, as many as fit)
    and CFS resumes.
    ``warm`` (test entry state, as in the oracle's sim.run): trace ids that
    arrive with prefill done (decode phase, g = 1, ctx = P) and their image
    already paged out (alloc + swap_out before iteration 0, not logged).
    ``max_iters`` stops after that many iterations.
    """
    pending = sorted(trace, key=lambda x: (x[1], x[0]))
    pi = 0
    log: List[tuple] = []
    i = 0
    blocks_out = blocks_in = 0
    swap_calls = []
    reclaimed = relent = False
    swapped_at = {}          # pid -> arena of its image
    warm = set(warm)
    for rid, _, P, _ in pending:
        if rid in warm:
            ctx.alloc_blocks(rid, -(-P // ctx.bs), decode_stream)
            ctx.swap_out([rid], swap_stream)
            swapped_at[rid] = ctx.query(rid)[1]
    while max_iters is None or i < max_iters:
        t = sched.vclock()
        while pi < len(pending) and pending[pi][1] <= t:
            rid, a, P, O = pending[pi]
            sched.add(rid, a, P, O)
            if rid in warm:
                sched.set_state(rid, 1, P, 1, P)
            pi += 1
        if elastic is not None and sched.stats()[0] > 0:
            if not reclaimed and t >= elastic["t_reclaim"]:
                peer = sorted(p for p, loc in swapped_at.items() if loc == aqua.LOC_PEER)
                tk = ctx.reclaim(swap_stream)
                moved = []
                for p in peer:
                    q = ctx.query(p, with_ids=True)
                    swapped_at[p] = q[1]
                    moved.append((p, tuple(q[3])))
                swap_calls.append(("reclaim", sum(len(x[1]) for x in moved), tk, time.perf_counter()))
                sched.set_policy(1)
                reclaimed = True
                if record_log:
                    log.append(("reclaim", i, tuple(moved)))
                    log.append(("policy", i, "fcfs"))
            elif reclaimed and not relent and t >= elastic["t_relend"]:
                dev, base, nbytes = elastic["relend"]
                n = ctx.lend(dev, base, nbytes)
                relent = True
                back, room = [], n
                for p in sorted(p for p, loc in swapped_at.items() if loc == aqua.LOC_HOST):
                    k = ctx.query(p)[2]
                    if k > room:
                        break
                    back.append(p)
                    room -= k
                if record_log:
                    log.append(("relend", i, n))
                if back:
                    tk = ctx.migrate(back, aqua.LOC_PEER, swap_stream)
                    slots = []
                    for p in back:
                        q = ctx.query(p, with_ids=True)
                        swapped_at[p] = q[1]
                        slots.append(tuple(q[3]))
                    swap_calls.append(("migrate", sum(len(x) for x in slots), tk, time.perf_counter()))
                    if record_log:
                        log.append(("migrate", i, tuple(back), tuple(slots)))
                sched.set_policy(policy_after_relend)
                if record_log:
                    log.append(("policy", i, "cfs" if policy_after_relend == 0 else "fcfs"))
        res, outs, ins, work = sched.next()
        if not work:
            if pi >= len(pending):
                break
            sched.advance_to(pending[pi][1])
            continue
        if res and record_log:
            D, PF = sched.partition()
            log.append(("plan", i, tuple(D), tuple((p, t) for p, t in PF)))
        if outs and ins and exchange_stream is not None:
            if stream_sync:
                stream_sync("before_swap_out", 0)
            t0 = time.perf_counter()
            new, tko, tki = ctx.swap_exchange(outs, ins, swap_stream, exchange_stream, exchange_pieces)
            q = [ctx.query(p, with_ids=True) for p in outs]
            n_o = sum(x[2] for x in q)
            n_i = sum(len(x) for x in new)
            blocks_out += n_o
            blocks_in += n_i
            for p, x in zip(outs, q):
                swapped_at[p] = x[1]
            for p in ins:
                swapped_at.pop(p, None)
            swap_calls.append(("out", n_o, tko, t0))
            swap_calls.append(("in", n_i, tki, t0))
            if on_swap:
                on_swap("out", outs, tko, n_o)
            if stream_sync:
                stream_sync("after_swap_in", tki)
            if on_swap:
                on_swap("in", ins, tki, n_i)
            if record_log:
                log.append(("swap_out", tuple(outs), tuple((x[1], tuple(x[3])) for x in q)))
                log.append(("swap_in", tuple(ins), tuple(tuple(x) for x in new)))
            outs = ins = []
        if outs:
            if stream_sync:
                stream_sync("before_swap_out", 0)
            t0 = time.perf_counter()
            tk = ctx.swap_out(outs, swap_stream)
            q = [ctx.query(p, with_ids=True) for p in outs]
            for p, x in zip(outs, q):
                swapped_at[p] = x[1]
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
            for p in ins:
                swapped_at.pop(p, None)
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
        if fill_seed is not None and work:
            ctx.kv_fill_pattern_batch([w[0] for w in work], [w[1] for w in work], [w[1] + w[2] for w in work],
                                      fill_seed, decode_stream)
        if on_iteration:
            on_iteration(i, work)
        fin, _ = sched.commit()
        for pid in fin:
            swapped_at.pop(pid, None)
            ctx.free(pid, decode_stream)
            if record_log:
                log.append(("free", pid))
        i += 1
    return log, {"iters": i, "blocks_out": blocks_out, "blocks_in": blocks_in, "swap_calls": swap_calls,
                 "vclock": sched.vclock()}
