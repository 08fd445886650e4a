"""Pins for oracle/cfs.py and oracle/sim.py.

* the paper's Fig. 6 scenario as worked by SPEC, golden fixture;
* SPEC's degenerate cases;
* brute-force round robin: n equal decode prompts, memory for m, must run in
  windows of m taken cyclically from the arrival-ordered queue, every k
  iterations (a deque-rotation model, not the oracle's sort);
* exhaustive tiny instances: least-service modulo memory, token
  budget <= b, memory feasibility;
* CFS == FCFS when there is no memory contention;
* no starvation within k*ceil(n/m) reschedules.
"""
import collections
import itertools
import json
import math
import os

import pytest

from oracle import cfs, sim
from oracle.cfs import DECODE, PREFILL, Req

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _fig6():
    g = json.load(open(os.path.join(GOLD, "cfs_fig6.json")))
    rs, names = [], {}
    for p in g["prompts"]:
        rs.append(Req(id=p["id"], arrival=p["arrival"], P=p["P"], O=p["O"], f=p["f"], g=p["g"],
                      ctx=p["ctx"], phase=DECODE if p["phase"] == "decode" else PREFILL))
        names[p["id"]] = p["name"]
    return g, rs, names


@pytest.mark.parametrize("variant", ["capacity3", "blocklevel"])
def test_fig6_worked_example(variant):
    g, rs, names = _fig6()
    v = g[variant]
    D, PF = cfs.plan(rs, g["b"], v["NB"], v["bs"])
    assert [names[i] for i in D] == v["decode"]
    assert [[names[i], t] for i, t in PF] == v["prefill"]
    # D starves in this plan ("D starves till A completes" under
    # FCFS); CFS serves it after k iterations -- see test below.


def test_fig6_d_runs_after_a_slice():
    """After one slice of k iterations of the Fig. 6 plan, D (no service)
    is scheduled and the most-served prompt A is displaced."""
    g, rs, names = _fig6()
    v = g["after_slice"]
    by = {r.id: r for r in rs}
    D, PF = cfs.plan(rs, g["b"], v["NB"], v["bs"])
    for _ in range(v["k"]):
        for i in D:
            by[i].ctx += 1
            by[i].g += 1
        for i, t in PF:
            r = by[i]
            if r.phase == PREFILL:
                t = min(t, r.P - r.f)
                r.f += t
                r.ctx += t
                if r.f == r.P:
                    r.phase, r.g = DECODE, 1
    assert (by[0].g, by[1].g, by[2].phase) == (58, 18, DECODE)
    D2, PF2 = cfs.plan(rs, g["b"], v["NB"], v["bs"])
    assert [names[i] for i in D2] == v["decode"]
    assert [[names[i], t] for i, t in PF2] == v["prefill"]
    before = {names[i] for i in D} | {names[i] for i, _ in PF}
    after = {names[i] for i in D2} | {names[i] for i, _ in PF2}
    assert sorted(before - after) == v["paged_out"]


def test_spec_degenerate_cases():
    rs = [Req(id=i, arrival=i, P=10, O=100, f=10, g=1 + i, ctx=10 + i, phase=DECODE) for i in range(5)]
    D, PF = cfs.plan(rs, 512, 1000, 16)
    assert D == [0, 1, 2, 3, 4] and PF == []
    one = [Req(id=9, arrival=0, P=100, O=10)]
    assert cfs.plan(one, 512, 1000, 16) == ([], [(9, 100)])


def test_r21_prefill_only_run_set_larger_than_b():
    """R21: with >= b prompts fitting, d = b and p = 0; without
    decode prompts the paper's "remaining slots in d are allocated to
    prompts in p" must still schedule prefill, else the plan is empty and
    the engine stalls (SPEC partition_batch: "empty plan only if nothing
    runnable").  Hand-executed: C = 5 prompts fit, d = min(4, 5) = 4,
    p = 0, D = [], the 4 spare slots walk the prefill order: prompt 0
    (least f, earliest arrival) takes min(4, 10) = 4 tokens."""
    rs = [Req(id=i, arrival=float(i), P=10, O=5) for i in range(5)]
    assert cfs.plan(rs, 4, 100, 16) == ([], [(0, 4)])
    # spare slots spill over prompts in prefill order: P = 3 each -> 3 + 1
    rs = [Req(id=i, arrival=float(i), P=3, O=5) for i in range(6)]
    assert cfs.plan(rs, 4, 100, 16) == ([], [(0, 3), (1, 1)])
    # two decode prompts and six prefill ones, b = 4: d = 4, D = [10, 11], 2 spare slots -> prefill
    dec = [Req(id=10 + i, arrival=float(i), P=16, O=9, f=16, g=1, ctx=16, phase=DECODE) for i in range(2)]
    assert cfs.plan(dec + rs, 4, 100, 16) == ([10, 11], [(0, 2)])
    # the memory test still applies: one block, a prompt with a 16-token KV cannot add tokens
    full = [Req(id=0, arrival=0.0, P=40, O=5, f=16, ctx=16)] + [Req(id=i, arrival=float(i), P=40, O=5)
                                                                  for i in range(1, 4)]
    assert cfs.plan(full, 2, 2, 16) == ([], [(1, 2)])


def test_plan_never_empty_while_a_prompt_fits():
    """SPEC S:275 as a property over random states: if some runnable prompt's
    KV plus one token fits the pool alone, the plan schedules something."""
    import random
    rnd = random.Random(5)
    for _ in range(3000):
        n = rnd.randint(1, 12)
        bs = rnd.choice([1, 4, 16])
        rs = []
        for i in range(n):
            P, O = rnd.randint(1, 200), rnd.randint(1, 40)
            if rnd.random() < 0.6:
                f = rnd.randint(0, P - 1)
                rs.append(Req(id=i, arrival=float(rnd.randint(0, 4)), P=P, O=O, f=f, ctx=f))
            else:
                g = rnd.randint(1, O)
                rs.append(Req(id=i, arrival=float(rnd.randint(0, 4)), P=P, O=O, f=P, g=g, ctx=P + g - 1,
                              phase=DECODE))
        b = rnd.choice([1, 2, 3, 8, 64])
        NB = rnd.randint(1, 60)
        D, PF = cfs.plan(rs, b, NB, bs)
        order = sorted((r for r in rs if r.phase == PREFILL), key=lambda r: (r.f, r.arrival, r.id)) + \
            sorted((r for r in rs if r.phase == DECODE), key=lambda r: (r.g, r.arrival, r.id))
        if cfs.need(order[0], 1, bs) <= NB:
            assert D or PF, (b, NB, bs, rs)


def _rotation_windows(n, m, slices):
    q = collections.deque(range(n))
    out = []
    for _ in range(slices):
        out.append(set(list(q)[:m]))
        q.rotate(-m)
    return out


@pytest.mark.parametrize("n,m,k", [(n, m, k) for n in range(1, 7) for m in range(1, n + 1) for k in (1, 2, 3)])
def test_bruteforce_round_robin(n, m, k):
    """n decode prompts with 8 tokens of context, bs=64 (one block each for
    the whole horizon), NB=m: the resident set must follow the rotating
    queue, and each reschedule swaps exactly the symmetric difference."""
    rs = [Req(id=i, arrival=float(i), P=8, O=10 ** 6, f=8, g=1, ctx=8, phase=DECODE) for i in range(n)]
    want = _rotation_windows(n, m, 30 // k + 1)
    prev = set()
    for s in range(len(want)):
        D, PF = cfs.plan(rs, 512, m, 64)
        assert PF == []
        assert set(D) == want[s], (s, D)
        assert len(prev - set(D)) == len(set(D) - prev) or not prev
        prev = set(D)
        for _ in range(k):
            for r in rs:
                if r.id in D:
                    r.ctx += 1
                    r.g += 1
        assert all(r.ctx <= 64 for r in rs)


def _sim_round_robin_expected(order, m, k, horizon):
    """Deque-rotation model of the whole reschedule loop (SURVEY
    C-9), independent of oracle.sim: `order` = pids in arrival order.  At
    every i = s*k the plan is the window of m at the head of the queue (in
    queue order), the queue is rotated by m, page_out = previous window
    minus this one and page_in = this window minus the previous one, both
    in arrival order; every iteration decodes the window, one token each."""
    pos = {pid: j for j, pid in enumerate(order)}
    q = collections.deque(order)
    served = {pid: 0 for pid in order}
    log = []
    prev = []
    win = []
    for i in range(horizon):
        if i % k == 0:
            win = list(q)[:m]
            q.rotate(-m)
            log.append(("plan", i, tuple(win), ()))
            out = sorted(set(prev) - set(win), key=pos.get)
            inn = sorted(set(win) - set(prev), key=pos.get)
            if out:
                log.append(("swap_out", tuple(out)))
            if inn:
                log.append(("swap_in", tuple(inn)))
            prev = win
        log.append(("iter", i, tuple((pid, 8 + served[pid], 1) for pid in win)))
        for pid in win:
            served[pid] += 1
    return log


@pytest.mark.parametrize("ids", ["arrival", "reversed"])
@pytest.mark.parametrize("n,m,k", [(n, m, k) for n in range(1, 7) for m in range(1, n + 1) for k in (1, 2, 3)])
def test_sim_reschedule_round_robin(n, m, k, ids):
    """C-9 pin of oracle.sim.run itself (not cfs.plan): n decode-only prompts
    (8 tokens of KV, bs=64 -> one block for the whole 30-iteration horizon,
    O huge), NB=m.  The full call log must equal the deque-rotation model:
    plans exactly at i = 0 (mod k), page lists = set differences of
    consecutive windows sorted by arrival, one block per paged prompt.  With
    ids in reverse arrival order, sorting by id instead of (arrival, id)
    fails; so does any off-by-one in the k cadence."""
    order = list(range(n)) if ids == "arrival" else [100 + n - 1 - j for j in range(n)]
    trace = [(pid, -100.0 + j, 8, 10 ** 6) for j, pid in enumerate(order)]
    H = 30
    res = sim.run(trace, sim.SimConfig(NB=m, bs=64, b=512, k=k, host_slots=64, max_iters=H), warm=order)
    want = _sim_round_robin_expected(order, m, k, H)
    got = []
    for e in res.log:
        if e[0] in ("swap_out", "swap_in"):
            # one block / one slot per paged prompt (per-reschedule block counts)
            per = [len(x[1]) for x in e[2]] if e[0] == "swap_out" else [len(x) for x in e[2]]
            assert per == [1] * len(e[1]), e
            got.append((e[0], e[1]))
        else:
            got.append(e)
    assert got == want
    assert res.blocks_out == sum(len(e[1]) for e in want if e[0] == "swap_out")
    assert res.blocks_in == sum(len(e[1]) for e in want if e[0] == "swap_in")


def _grid():
    states = []
    for phase, f, g, ctx in [(PREFILL, 0, 0, 0), (PREFILL, 20, 0, 20), (PREFILL, 40, 0, 40),
                             (DECODE, 50, 1, 50), (DECODE, 50, 5, 54), (DECODE, 50, 9, 58)]:
        states.append((phase, f, g, ctx))
    return states


@pytest.mark.parametrize("NB", [2, 4, 7, 100])
@pytest.mark.parametrize("b", [1, 3, 33, 512])
def test_exhaustive_plan_properties(NB, b):
    bs = 16
    grid = _grid()
    for n in (1, 2, 3):
        for combo in itertools.product(range(len(grid)), repeat=n):
            rs = []
            for i, gi in enumerate(combo):
                phase, f, g, ctx = grid[gi]
                rs.append(Req(id=i, arrival=float((i * 7) % 3), P=50, O=20, f=f, g=g, ctx=ctx, phase=phase))
            D, PF = cfs.plan(rs, b, NB, bs)
            by = {r.id: r for r in rs}
            toks = {i: 1 for i in D}
            toks.update(dict(PF))
            # budget and no duplicates
            assert sum(toks.values()) <= b
            assert len(toks) == len(D) + len(PF)
            # memory feasibility (R11)
            assert sum(cfs.need(by[i], t, bs) for i, t in toks.items()) <= NB
            # tokens positive and prefill bounded by the prompt
            for i, t in PF:
                assert 0 < t <= by[i].P - by[i].f and by[i].phase == PREFILL
            # least service: every scheduled decode precedes every
            # unscheduled one in (g, arrival, id); likewise prefill in f
            key_d = lambda r: (r.g, r.arrival, r.id)
            key_p = lambda r: (r.f, r.arrival, r.id)
            sd = [by[i] for i in D]
            ud = [r for r in rs if r.phase == DECODE and r.id not in toks]
            assert all(key_d(s) < key_d(u) for s in sd for u in ud)
            sp = [by[i] for i, _ in PF]
            up = [r for r in rs if r.phase == PREFILL and r.id not in toks]
            assert all(key_p(s) < key_p(u) for s in sp for u in up)
            # d upper bound: the decode count never exceeds b
            assert len(D) <= b


def _toy_trace(n=12, gap=0.05, seed=3):
    import random
    rnd = random.Random(seed)
    return [(i, i * gap, rnd.randint(1, 300), rnd.randint(1, 40)) for i in range(n)]


def test_cfs_equals_fcfs_without_contention():
    """P:985 'behavior of CFS is identical to FCFS when there is no memory
    contention': with ample memory CFS never pages; with one prompt at a
    time the iteration logs coincide exactly."""
    tr = _toy_trace()
    r = sim.run(tr, sim.SimConfig(NB=10 ** 6, lender_slots=100))
    assert r.blocks_out == 0 and r.blocks_in == 0
    assert not [e for e in r.log if e[0] in ("swap_out", "swap_in")]
    serial = [(i, i * 100.0, 100 + 13 * i, 5 + i) for i in range(5)]
    a = sim.run(serial, sim.SimConfig(NB=10 ** 6, policy="cfs"))
    b = sim.run(serial, sim.SimConfig(NB=10 ** 6, policy="fcfs"))
    it = lambda res: [e for e in res.log if e[0] in ("iter", "alloc", "free")]
    assert [e[1:] if e[0] != "iter" else e[2] for e in it(a)] == \
           [e[1:] if e[0] != "iter" else e[2] for e in it(b)]


@pytest.mark.parametrize("k", [1, 4, 8])
def test_no_starvation_and_conservation(k):
    """every runnable prompt is scheduled within k*ceil(n/m)
    reschedule intervals; swapped bytes conserved (blocks out == in once all
    finish); the pool invariants hold (checked inside sim.run)."""
    tr = [(i, 0.0, 40, 30) for i in range(6)]          # all arrive together
    NB = 9                                               # ~2-3 prompts fit (bs=16)
    res = sim.run(tr, sim.SimConfig(NB=NB, bs=16, b=64, k=k, lender_slots=64))
    assert set(res.finish) == set(range(6))
    assert res.blocks_out == res.blocks_in
    first_iter = {}
    for e in res.log:
        if e[0] == "iter":
            for pid, _, t in e[2]:
                first_iter.setdefault(pid, e[1])
    # at least one prompt always fits (m >= 1) and a reschedule happens at
    # least every k iterations, so first service is within k*ceil(n/1)
    assert max(first_iter.values()) <= k * math.ceil(6 / 1)
    plans = [e for e in res.log if e[0] == "plan"]
    assert plans and plans[0][1] == 0


def test_sim_determinism_and_paging_happens():
    from workloads import burst_trace
    tr = burst_trace(seed=1, burst_s=6.0, tail_s=2.0, prompt=(400, 0.8, 1, 1024), output=(40, 0.7, 1, 200))
    cfg = sim.SimConfig(NB=160, bs=16, lender_slots=400)
    a = sim.run(tr, cfg)
    b = sim.run(tr, cfg)
    assert a.log == b.log
    assert a.blocks_out > 0 and a.blocks_out == a.blocks_in
    assert set(a.finish) == {t[0] for t in tr}


# ------------------------------------------------------------- FCFS (R18)
def test_fcfs_admission_in_arrival_order_and_projection():
    """Pure FCFS: first service follows arrival order and
    the admitted projections never exceed the pool; it never pages."""
    tr = [(i, 0.05 * i, 50 + 37 * (i % 5), 20 + 11 * (i % 3)) for i in range(12)]
    NB = 40
    r = sim.run(tr, sim.SimConfig(NB=NB, b=128, policy="fcfs", lender_slots=100))
    assert not [e for e in r.log if e[0] in ("swap_out", "swap_in", "plan")]
    first = []
    for e in r.log:
        if e[0] == "iter":
            for pid, _, _ in e[2]:
                if pid not in first:
                    first.append(pid)
    assert first == sorted(first)                       # arrival order == id order here
    # projection bound: at any iteration the prompts holding KV fit their full need
    live = set()
    for e in r.log:
        if e[0] == "alloc":
            live.add(e[1])
        elif e[0] == "free":
            live.discard(e[1])
        elif e[0] == "iter":
            assert sum(-(-(tr[p][2] + tr[p][3]) // 16) for p in live) <= NB


def test_fallback_keeps_residents_and_evicts_latest_arrival():
    """CFS -> FCFS fallback (R18): the residents at the switch stay
    admitted; when they outgrow the pool the latest-arrived resident is the
    one paged out; while in fallback there is no CFS replanning and every
    page-out goes to DRAM."""
    tr = [(i, 0.01 * i, 40, 300) for i in range(8)]
    r = sim.run(tr, sim.SimConfig(NB=40, b=64, lender_slots=400, host_slots=2000, elastic=(0.5, 1e9),
                                  relend_slots=400))
    i_sw = [k for k, e in enumerate(r.log) if e[0] == "policy"][0]
    # residents just before the switch
    res = set()
    for e in r.log[:i_sw]:
        if e[0] == "alloc":
            res.add(e[1])
        elif e[0] == "swap_out":
            res -= set(e[1])
        elif e[0] == "swap_in":
            res |= set(e[1])
        elif e[0] == "free":
            res.discard(e[1])
    outs = [e for e in r.log[i_sw:] if e[0] == "swap_out"]
    assert outs, "the scenario must overflow"
    # every fallback eviction is the latest-arrived resident at that moment
    cur = set(res)
    for e in r.log[i_sw:]:
        if e[0] == "swap_out":
            (victim,) = e[1]
            assert victim == max(cur, key=lambda p: (tr[p][1], p))
            assert all(loc == 2 for loc, _ in e[2])      # to DRAM: the lender is gone
            cur.discard(victim)
        elif e[0] == "swap_in":
            cur |= set(e[1])
        elif e[0] == "alloc":
            cur.add(e[1])
        elif e[0] == "free":
            cur.discard(e[1])
        assert e[0] != "plan"


def test_relend_moves_back_lowest_pids_that_fit():
    """NEXT-1 re-offer (P:1086 'moves the offloaded tensors of the consumer
    back to the producer's GPU'): after the lender returns, host images move
    back in ascending pid while they fit, into the lowest slots; CFS resumes
    with a fresh plan."""
    tr = [(i, 0.01 * i, 40, 300) for i in range(8)]
    r = sim.run(tr, sim.SimConfig(NB=40, b=64, lender_slots=400, host_slots=2000, elastic=(2.0, 3.0),
                                  relend_slots=7))
    kinds = [e[0] for e in r.log]
    assert len(r.log[kinds.index("reclaim")][2]) == 3       # three images were on the lender
    i_rel = kinds.index("relend")
    assert r.log[i_rel][2] == 7
    # host images just before the re-offer
    host, sizes = {}, {}
    for e in r.log[:i_rel]:
        if e[0] == "swap_out":
            for pid, (loc, sl) in zip(e[1], e[2]):
                host[pid] = loc == 2
                sizes[pid] = len(sl)
        elif e[0] == "reclaim":
            for pid, sl in e[2]:
                host[pid] = True
        elif e[0] in ("swap_in",):
            for pid in e[1]:
                host.pop(pid, None)
        elif e[0] == "free":
            host.pop(e[1], None)
    on_host = sorted(p for p, h in host.items() if h)
    want, room = [], 7
    for p in on_host:
        if sizes[p] > room:
            break
        want.append(p)
        room -= sizes[p]
    mig = [e for e in r.log[i_rel:i_rel + 3] if e[0] == "migrate"]
    assert want and on_host[len(want):], "scenario must move some images back and leave one"
    if want:
        assert list(mig[0][2]) == want
        flat = [s for sl in mig[0][3] for s in sl]
        assert flat == list(range(len(flat)))           # lowest slots of the fresh lender
    else:
        assert not mig
    assert ("policy", r.log[i_rel][1], "cfs") in r.log[i_rel:i_rel + 4]
    assert r.log[i_rel + (2 if mig else 1) + 1][0] == "plan"   # a fresh CFS plan right after


def test_replay_bytes_keeps_every_prompt_closed_form():
    """sim.replay_bytes (the bytes mode of the trace driver) pinned to the
    closed-form content (C-11, invariant I8): after every 6th iteration, each
    prompt it ran holds exactly its pattern words for all its KV tokens,
    across any number of preemptions; the call results equal the log."""
    from oracle import kvpool as kp
    from oracle import pattern
    from workloads import burst_trace, kv_random_bytes
    tr = burst_trace(seed=3, burst_s=4.0, tail_s=2.0, prompt=(120, 0.8, 1, 400), output=(20, 0.7, 1, 80))
    cfg = sim.SimConfig(NB=60, bs=16, lender_slots=120, host_slots=400, k=4)
    res = sim.run(tr, cfg)
    assert res.blocks_out > 0
    lay = kp.Layout(L=2, bs=16, H=2, D=8, e=2, NB=60)
    pool = kp.Pool(lay, [kv_random_bytes(lay.layer_bytes, seed=l) for l in range(2)])
    pool.lend(kp.LOC_PEER, 120 * lay.U, kv_random_bytes(120 * lay.U, seed=5))
    pool.lend(kp.LOC_HOST, 400 * lay.U, kv_random_bytes(400 * lay.U, seed=6))
    iters = {e[1]: e[2] for e in res.log if e[0] == "iter"}
    checked = []

    def check(i):
        if i % 6:
            checked.append(i)
            return
        for pid, ctx0, t in iters[i]:
            assert pattern.check_tokens(pool, pid, ctx0 + t, seed=3), (i, pid)
        checked.append(i)

    sim.replay_bytes(res.log, pool, 3, on_iter=check)
    assert len(checked) == res.iters


# ------------------------------------------- pins added by the mutation check
# Each case below is hand-executed from the paper / SPEC text (expected values
# derived on paper, not by running the oracle).  They kill the mutants that
# scripts/oracle_mutants.py found surviving the earlier pins.

def test_step3_decode_walk_stops_at_the_first_prompt_that_does_not_fit():
    """R12, "Aqua stops filling the batch if the GPU's memory is
    exhausted".  NB=4, bs=16, b=20.  X prefill (P=40, nothing done); A decode
    (g=1, ctx=32: needs ceil(33/16)=3 blocks); B decode (g=2, ctx=15: 1 block).
    Step 1 walks X (1 block), A (3) -> 4 used, B does not fit: C=2, d=2,
    p=18.  Step 2: X gets 18 tokens = 2 blocks.  Step 3 (least generated
    first): A needs 3 more -> 5 > 4, the walk stops; B (which would fit) is
    NOT taken.  Step 4: the 2 unused decode slots go to X: 20 tokens, still
    2 blocks.  Plan: D = [], prefill [(X, 20)]."""
    X = Req(0, 0.0, 40, 5, 0, 0, 0, PREFILL)
    A = Req(1, 1.0, 16, 100, 16, 1, 32, DECODE)
    B = Req(2, 2.0, 15, 100, 15, 2, 15, DECODE)
    assert cfs.plan([X, A, B], 20, 4, 16) == ([], [(0, 20)])


def test_fcfs_plan_decodes_at_most_b_prompts():
    """SPEC fcfs_step: one decode token per admitted decode prompt
    in arrival order, within the batch budget b; nothing left for prefill."""
    rs = [Req(i, float(i), 8, 100, 8, 1, 8, DECODE) for i in (4, 2, 0, 3, 1)]
    assert cfs.fcfs_plan(rs, 3) == ([0, 1, 2], [])
    assert cfs.fcfs_plan(rs, 7) == ([0, 1, 2, 3, 4], [])


def test_sim_reschedules_when_a_request_completes():
    """P:836-837 "Aqua reschedules the batch every k iterations OR WHEN A
    REQUEST COMPLETES".  Three decode-only prompts already paged out (8 tokens
    of KV, bs=64: one block each), NB=2, k=1000 (no time-slice reschedule in
    the horizon).  Prompt 0 has O=3: it is at g=1, decodes at iterations 0 and
    1 and completes after iteration 1.  The plan made at iteration 0 holds
    {0, 1} (all g=1, arrival order); at iteration 2 a reschedule must page in
    prompt 2 (least generated, g=1) beside prompt 1 (g=3)."""
    tr = [(0, -3.0, 8, 3), (1, -2.0, 8, 10 ** 6), (2, -1.0, 8, 10 ** 6)]
    r = sim.run(tr, sim.SimConfig(NB=2, bs=64, b=512, k=1000, host_slots=64, max_iters=6), warm=[0, 1, 2])
    plans = [(e[1], e[2]) for e in r.log if e[0] == "plan"]
    assert plans == [(0, (0, 1)), (2, (2, 1))]
    assert ("swap_in", (2,), ((0,),)) in r.log           # block 0, freed by prompt 0
    iters = {e[1]: tuple(p for p, _, _ in e[2]) for e in r.log if e[0] == "iter"}
    assert iters == {0: (0, 1), 1: (0, 1), 2: (2, 1), 3: (2, 1), 4: (2, 1), 5: (2, 1)}


def test_sim_virtual_clock_closed_form():
    """S:233 iteration time t = 20 ms + 40 us x tokens; R15 first token at the
    end of prefill (g = 1), finish when g == O.  One request alone (P=100,
    O=4, memory ample): iteration 0 prefills 100 tokens (24 ms) -> TTFT
    0.024 s; then O-1 = 3 decode iterations of one token (20.04 ms each) ->
    finish 0.024 + 3 x 0.02004 = 0.08412 s, 4 iterations in all."""
    r = sim.run([(0, 0.0, 100, 4)], sim.SimConfig(NB=1000))
    assert r.iters == 4
    assert r.ttft[0] == pytest.approx(0.024, rel=1e-12)
    assert r.finish[0] == pytest.approx(0.024 + 3 * 0.02004, rel=1e-12)


def test_fcfs_admits_while_the_projection_fits_exactly():
    """S:297-305 "admit ... while the sum of full projections ceil((P+O)/bs)
    fits NB": two requests of P=16, O=16 (2 blocks each at bs=16) fill NB=4
    exactly, so both run in iteration 0 (16 prefill tokens each)."""
    r = sim.run([(0, 0.0, 16, 16), (1, 0.0, 16, 16)], sim.SimConfig(NB=4, bs=16, policy="fcfs"))
    it0 = next(e for e in r.log if e[0] == "iter")
    assert it0 == ("iter", 0, ((0, 0, 16), (1, 0, 16)))


def test_reoffer_stops_at_the_first_image_that_does_not_fit():
    """R22 (NEXT-1 re-offer): host images move back in ascending pid
    WHILE they fit the re-offered lender -- the walk stops at the first that
    does not (R12's rule applied to the re-offer), it does not skip ahead.
    Scenario with unequal image sizes where the two readings differ: the host
    holds pids 3, 4, 5, ... with 6, 11, ... blocks, the re-offer has 12 slots:
    pid 3 moves (6 <= 12), pid 4 (11 > 6 left) stops the walk, so a later
    6-block image that would fit stays on the host."""
    Ps = (40, 200, 40, 40, 120, 40, 40, 40)
    tr = [(i, 0.01 * i, Ps[i], 300) for i in range(8)]
    r = sim.run(tr, sim.SimConfig(NB=40, b=64, lender_slots=400, host_slots=2000, elastic=(2.0, 3.0),
                                  relend_slots=12))
    kinds = [e[0] for e in r.log]
    i_rel = kinds.index("relend")
    host, sizes = {}, {}
    for e in r.log[:i_rel]:
        if e[0] == "swap_out":
            for pid, (loc, sl) in zip(e[1], e[2]):
                host[pid] = loc == 2
                sizes[pid] = len(sl)
        elif e[0] == "reclaim":
            for pid, sl in e[2]:
                host[pid] = True
        elif e[0] == "swap_in":
            for pid in e[1]:
                host.pop(pid, None)
        elif e[0] == "free":
            host.pop(e[1], None)
    on_host = sorted(p for p, h in host.items() if h)
    stop, skip, room_a, room_b = [], [], 12, 12
    for p in on_host:
        if sizes[p] <= room_b:
            skip.append(p)
            room_b -= sizes[p]
    for p in on_host:
        if sizes[p] > room_a:
            break
        stop.append(p)
        room_a -= sizes[p]
    assert stop != skip, "the scenario must tell the two readings apart"
    mig = next(e for e in r.log[i_rel:] if e[0] == "migrate")
    assert list(mig[2]) == stop
