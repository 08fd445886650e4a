"""Oracle: metadata-mode trace driver (C3) -- CFS reschedule + paging calls.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper, Sec. 7: "For simplicity, we measure time slices as the
number of inference iterations, as each iteration of a given batch size
takes the same time. Aqua reschedules the batch every k iterations or when a
request completes, paging out prompts that are not a part of the next batch
and paging in prompts that were not on the GPU."
SPEC reschedule S:279-287; iteration cost t = 20 ms + 40 us * tokens
 drives a VIRTUAL clock used only for admission, so the
schedule never depends on measured swap speed.

Readings: R8 k = 8 by default; R11 an extra reschedule trigger
when the current plan's next iteration no longer fits in NB (and when the
plan has no work left); R13 page_out = every resident prompt not in the
plan (literal); R14 a prompt preempted mid-prefill keeps its partial KV.

Iteration semantics (R15): a prefill prompt scheduled for t tokens stores t
KV tokens (ctx += t, f += t); when f reaches P it emits its first token
(g = 1) and idles until the next plan.  A decode prompt stores the
KV of its last token and emits one more (ctx += 1, g += 1); it finishes when
g == O.  Before an iteration each scheduled prompt is grown to
ceil((ctx + t) / bs) blocks with alloc_blocks, in plan order.

The driver emits the exact call log the GPU run must reproduce:
  ("swap_out", pids, [(loc, slots), ...])   ("swap_in", pids, [ids, ...])
  ("alloc", pid, ids)    ("free", pid)    ("iter", i, [(pid, ctx0, t), ...])
  ("plan", i, decode_ids, [(pid, tokens), ...])
  ("reclaim", i, ((pid, slots), ...))   ("relend", i, nslots)
  ("migrate", i, pids, (slots, ...))    ("policy", i, "fcfs"|"cfs")

NEXT-1 elasticity: reclaim moves every lender image
to DRAM and FCFS takes over; a re-offer moves DRAM images back in ascending
pid while they fit, stopping at the first that does not (R22), then CFS
replans.

FCFS (R18; SPEC fcfs_step S:297-305, fallback S:306-313): requests are
admitted in (arrival, id) order while the sum of their full projections
ceil((P+O)/bs) fits NB; a swapped prompt is paged in when admitted; the
plan decodes every admitted decode prompt, then prefills in arrival order.
When FCFS takes over from CFS (fallback) the admitted set starts as the
resident prompts; if their growth no longer fits, the latest-arrived
admitted resident is paged out (the vLLM FCFS preemption order).
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Sequence, Tuple

from . import cfs
from .cfs import DECODE, PREFILL, Req
from .kvpool import LOC_HOST, LOC_PEER, RESIDENT, SWAPPED, Layout, Pool


@dataclasses.dataclass
class SimConfig:
    NB: int
    bs: int = 16
    b: int = 512
    k: int = 8
    policy: str = "cfs"            # "cfs" or "fcfs"
    lender_slots: int = 0          # 0 -> no peer lender (DRAM only)
    host_slots: int = 1 << 14
    t_base: float = 0.020
    t_token: float = 40e-6
    max_iters: int = 10_000_000
    # NEXT-1 elasticity: the lender reclaims its
    # memory at virtual time elastic[0] and re-offers relend_slots at
    # elastic[1]; while the images sit in DRAM the engine runs FCFS
    elastic: Optional[Tuple[float, float]] = None
    relend_slots: int = 0


@dataclasses.dataclass
class SimResult:
    log: List[tuple]
    ttft: Dict[int, float]
    finish: Dict[int, float]
    iters: int
    blocks_out: int
    blocks_in: int
    vclock: float
    timeline: List[Tuple[float, int]]      # (virtual time at iteration start, blocks owned)


def run(trace: Sequence[Tuple[int, float, int, int]], cfg: SimConfig,
        warm: Sequence[int] = ()) -> SimResult:
    """trace = [(id, arrival_s, prompt_tokens, output_tokens)] sorted by
    (arrival, id).

    warm (test entry state, not a workload feature): trace ids that arrive
    with their prefill already done (f = ctx = P, g = 1, phase DECODE) and
    their KV image already paged out, as after an earlier preemption (the
    decode-only round-robin instances of SURVEY C-9).  Their images are
    placed before iteration 0 by alloc_blocks + swap_out, one prompt at a
    time in trace order; nothing is logged for this setup."""
    lay = Layout(L=1, bs=cfg.bs, H=1, D=8, e=2, NB=cfg.NB)   # metadata only
    pool = Pool(lay)
    if cfg.lender_slots > 0:
        pool.lend(LOC_PEER, cfg.lender_slots * lay.U)
    if cfg.host_slots > 0:
        pool.lend(LOC_HOST, cfg.host_slots * lay.U)

    pending = sorted(trace, key=lambda x: (x[1], x[0]))
    pi = 0
    warm = set(warm)
    for rid, _, P, _ in pending:
        if rid in warm:
            pool.alloc_blocks(rid, -(-P // lay.bs))
            pool.swap_out([rid])
    run_set: Dict[int, Req] = {}
    log: List[tuple] = []
    ttft: Dict[int, float] = {}
    finish: Dict[int, float] = {}
    admitted_fcfs: List[int] = []           # FCFS: admitted in arrival order
    t = 0.0
    i = 0
    plan = None
    last = 0
    finished_prev = False
    blocks_out = blocks_in = 0
    mode = cfg.policy
    reclaimed = relent = False
    timeline: List[Tuple[float, int]] = []

    def resident(pid):
        p = pool.prompts.get(pid)
        return p is not None and p.state == RESIDENT

    def this_iter_tokens(plan_):
        D, PF = plan_
        out = []
        for pid in D:
            r = run_set.get(pid)
            if r is not None and r.phase == DECODE:
                out.append((pid, 1))
        for pid, a in PF:
            r = run_set.get(pid)
            if r is not None and r.phase == PREFILL:
                out.append((pid, min(a, r.P - r.f)))
        return out

    def fits(work, leaving=()):
        tok = dict(work)
        tot = 0
        for pid, p in pool.prompts.items():
            if p.state == RESIDENT and pid not in leaving:
                tot += cfs.need(run_set[pid], tok.get(pid, 0), lay.bs)
        for pid, tt in work:
            if not resident(pid):
                tot += cfs.need(run_set[pid], tt, lay.bs)
        return tot <= lay.NB

    while (pi < len(pending) or run_set) and i < cfg.max_iters:
        while pi < len(pending) and pending[pi][1] <= t:
            rid, a, P, O = pending[pi]
            run_set[rid] = Req(id=rid, arrival=a, P=P, O=O)
            if rid in warm:
                run_set[rid] = Req(id=rid, arrival=a, P=P, O=O, f=P, g=1, ctx=P, phase=DECODE)
            pi += 1
        if not run_set:
            t = pending[pi][1]          # idle: jump to the next arrival
            plan = None
            continue

        if cfg.elastic is not None:
            if not reclaimed and t >= cfg.elastic[0]:
                res = pool.reclaim()
                log.append(("reclaim", i, tuple((pid, tuple(sl)) for pid, sl in res)))
                reclaimed = True
                mode = "fcfs"
                admitted_fcfs[:] = [pid for pid in sorted(run_set, key=lambda x: (run_set[x].arrival, x))
                                    if resident(pid)]
                log.append(("policy", i, "fcfs"))
            elif reclaimed and not relent and t >= cfg.elastic[1]:
                n = pool.lend(LOC_PEER, cfg.relend_slots * lay.U)
                log.append(("relend", i, n))
                relent = True
                back, room = [], n
                for pid in sorted(pid for pid, p in pool.prompts.items()
                                  if p.state == SWAPPED and p.location == LOC_HOST):
                    k = len(pool.prompts[pid].slots)
                    if k > room:
                        break
                    back.append(pid)
                    room -= k
                if back:
                    res = pool.migrate(back, LOC_PEER)
                    log.append(("migrate", i, tuple(back), tuple(tuple(sl) for _, sl in res)))
                mode = cfg.policy
                admitted_fcfs.clear()
                plan = None
                log.append(("policy", i, mode))

        if mode == "fcfs":
            # admission: full projection must fit, head-of-line
            proj = sum(-(-(run_set[x].P + run_set[x].O) // lay.bs) for x in admitted_fcfs)
            page_in = []
            for r in sorted(run_set.values(), key=lambda r: (r.arrival, r.id)):
                if r.id in admitted_fcfs:
                    continue
                n = -(-(r.P + r.O) // lay.bs)
                if proj + n > lay.NB:
                    break
                proj += n
                admitted_fcfs.append(r.id)
                if r.id in pool.prompts and pool.prompts[r.id].state == SWAPPED:
                    page_in.append(r.id)
            if page_in:
                res = pool.swap_in(page_in)
                blocks_in += sum(len(x) for x in res)
                log.append(("swap_in", tuple(page_in), tuple(tuple(x) for x in res)))
            plan = cfs.fcfs_plan([run_set[x] for x in admitted_fcfs], cfg.b)
            work = this_iter_tokens(plan)
            leaving = []
            while work and not fits(work, leaving):
                # overflow after a fallback: preempt the latest-arrived
                # resident until the iteration fits; the victims leave in one
                # call, latest arrival first (R18)
                victims = [x for x in admitted_fcfs if resident(x)]
                victim = max(victims, key=lambda x: (run_set[x].arrival, x))
                admitted_fcfs.remove(victim)
                leaving.append(victim)
                plan = cfs.fcfs_plan([run_set[x] for x in admitted_fcfs], cfg.b)
                work = this_iter_tokens(plan)
            if leaving:
                res = pool.swap_out(leaving)
                blocks_out += sum(len(s_) for _, _, s_ in res)
                log.append(("swap_out", tuple(leaving), tuple((loc, tuple(s_)) for _, loc, s_ in res)))
            if not work:
                raise RuntimeError("FCFS: the head-of-line prompt can never fit the pool")
        else:
            work = this_iter_tokens(plan) if plan is not None else []
            if (plan is None or i - last >= cfg.k or finished_prev or not work
                    or not fits(work)):
                plan = cfs.plan(list(run_set.values()), cfg.b, lay.NB, lay.bs)
                last = i
                log.append(("plan", i, tuple(plan[0]), tuple(plan[1])))
                in_plan = set(plan[0]) | {pid for pid, _ in plan[1]}
                key = lambda pid: (run_set[pid].arrival, pid)
                page_out = sorted((pid for pid in run_set if resident(pid) and pid not in in_plan), key=key)
                page_in = sorted((pid for pid in in_plan
                                  if pid in pool.prompts and pool.prompts[pid].state == SWAPPED), key=key)
                if page_out:
                    res = pool.swap_out(page_out)
                    blocks_out += sum(len(s) for _, _, s in res)
                    log.append(("swap_out", tuple(page_out), tuple((loc, tuple(s)) for _, loc, s in res)))
                if page_in:
                    res = pool.swap_in(page_in)
                    blocks_in += sum(len(x) for x in res)
                    log.append(("swap_in", tuple(page_in), tuple(tuple(x) for x in res)))
                work = this_iter_tokens(plan)
                if not work:
                    raise RuntimeError("empty plan with runnable prompts (pool too small)")

        # grow block tables in plan order, then run the iteration
        for pid, tt in work:
            r = run_set[pid]
            have = len(pool.prompts[pid].blocks) if pid in pool.prompts else 0
            n = cfs.need(r, tt, lay.bs) - have
            if n > 0:
                ids = pool.alloc_blocks(pid, n)
                log.append(("alloc", pid, tuple(ids)))
        log.append(("iter", i, tuple((pid, run_set[pid].ctx, tt) for pid, tt in work)))
        timeline.append((t, lay.NB - len(pool.free)))
        total = sum(tt for _, tt in work)
        t += cfg.t_base + cfg.t_token * total
        finished_prev = False
        for pid, tt in work:
            r = run_set[pid]
            if r.phase == PREFILL:
                r.f += tt
                r.ctx += tt
                if r.f == r.P:
                    r.phase, r.g = DECODE, 1
                    ttft[pid] = t - r.arrival
            else:
                r.ctx += 1
                r.g += 1
            if r.phase == DECODE and r.g >= r.O:
                finish[pid] = t - r.arrival
                pool.free_prompt(pid)
                log.append(("free", pid))
                del run_set[pid]
                if pid in admitted_fcfs:
                    admitted_fcfs.remove(pid)
                finished_prev = True
        i += 1
    pool.check_invariants()
    return SimResult(log, ttft, finish, i, blocks_out, blocks_in, t, timeline)


def replay_bytes(log: Sequence[tuple], pool: Pool, seed: int, on_iter=None) -> None:
    """Bytes mode of the trace driver (SURVEY 8(d) parity protocol, scaled-down
    C3): apply a call log that run() emitted to a bytes-mode Pool -- every
    paging call through the Pool's own operations (C-4 / C-5), and
    for each iteration the synthetic decode: tokens [ctx0, ctx0 + t) of each
    work item get their closed-form words (C-11).  Each call's result must
    equal the log's (ids, slots, locations).  on_iter(i) runs after iteration
    i's tokens are written.  Elastic entries (reclaim / relend / migrate) are
    not replayed."""
    from . import pattern
    for e in log:
        kind = e[0]
        if kind == "swap_out":
            res = pool.swap_out(e[1])
            assert tuple((loc, tuple(s)) for _, loc, s in res) == tuple(e[2]), e
        elif kind == "swap_in":
            res = pool.swap_in(e[1])
            assert tuple(tuple(x) for x in res) == tuple(e[2]), e
        elif kind == "alloc":
            ids = pool.alloc_blocks(e[1], len(e[2]))
            assert tuple(ids) == tuple(e[2]), e
        elif kind == "free":
            pool.free_prompt(e[1])
        elif kind == "iter":
            for pid, ctx0, t in e[2]:
                pattern.write_token_range(pool, pid, ctx0, ctx0 + t, seed)
            if on_iter is not None:
                on_iter(e[1])
        elif kind in ("plan", "policy"):
            pass
        else:
            raise NotImplementedError(f"bytes replay of {kind!r}")
