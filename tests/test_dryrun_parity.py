"""Host-logic parity on CPU: libaqua in AQUA_DRYRUN mode (bookkeeping and
descriptors, no CUDA) and the native CFS scheduler against the oracle.

Bit-exact (integers): ids, slots, locations, descriptors, error codes,
plans and whole call logs must be identical."""
import itertools
import json
import os
import random

import numpy as np
import pytest

from oracle import cfs as ocfs
from oracle import kvpool as kp
from oracle import sim as osim
from paper_2407_21255_b200 import aqua
from paper_2407_21255_b200.cfs import PHASE_DECODE, PHASE_PREFILL, POLICY_CFS, POLICY_FCFS, Scheduler
from paper_2407_21255_b200.driver import run_trace
from workloads import burst_trace

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FAKE = 1 << 40


def dry_ctx(L=2, bs=16, H=2, D=64, e=2, NB=40):
    S = bs * H * D * e
    ptrs = [FAKE + l * (1 << 32) for l in range(L)]
    return aqua.Ctx(aqua.DRYRUN, L, bs, H, D, e, NB, ptrs)


@pytest.mark.parametrize("variant", ["lender12", "lender8"])
def test_c1_script_dryrun(variant):
    g = json.load(open(os.path.join(GOLD, "c1_script.json")))
    v = g[variant]
    lay = g["layout"]
    c = dry_ctx(**lay)
    assert c.lend(0, FAKE * 2, v["lender_slots"] * c.U) == v["lender_slots"]
    if v.get("host_slots"):
        c.lend(aqua.HOST, FAKE * 3, v["host_slots"] * c.U)
    for p in range(g["prompts"]):
        assert c.alloc_blocks(p, g["blocks_per_prompt"]) == g["initial_ids"][str(p)]
    c.swap_out(g["swap_out"])
    b, s, l = c.last_descriptors()
    want_b, want_s, want_l = [], [], []
    for pid in g["swap_out"]:
        loc, slots = v["placement"][str(pid)]
        st, qloc, n, ids = c.query(pid, with_ids=True)
        assert st == aqua.SWAPPED and ids == slots
        assert qloc == {"peer": aqua.LOC_PEER, "host": aqua.LOC_HOST}[loc]
        want_b += g["initial_ids"][str(pid)]
        want_s += slots
        want_l += [qloc] * len(slots)
    assert (b, s, l) == (want_b, want_s, want_l)
    assert c.alloc_blocks(g["filler"]["pid"], g["filler"]["n"]) == g["filler"]["expected_ids"]
    new, _ = c.swap_in(g["swap_in"])
    for pid, ids in zip(g["swap_in"], new):
        assert ids == g["expected_swap_in_ids"][str(pid)]
    c.free(g["filler"]["pid"])
    assert c.counts()[0] == 40 - 32


def _apply(pool, c, op):
    """Run one op on the oracle and on the dry-run ctx; return both results."""
    name, arg = op
    res = []
    for side in ("oracle", "lib"):
        try:
            if name == "alloc":
                r = pool.alloc_blocks(*arg) if side == "oracle" else c.alloc_blocks(*arg)
            elif name == "adopt":
                r = pool.adopt_blocks(*arg) if side == "oracle" else c.adopt_blocks(*arg)
            elif name == "out":
                if side == "oracle":
                    r = [(loc, s) for _, loc, s in pool.swap_out(arg)]
                else:
                    c.swap_out(arg)
                    r = [(c.query(p)[1], c.query(p, with_ids=True)[3]) for p in arg]
            elif name == "in":
                r = pool.swap_in(arg) if side == "oracle" else c.swap_in(arg, cap=1 << 12)[0]
            elif name == "free":
                r = pool.free_prompt(arg) if side == "oracle" else c.free(arg)
            elif name == "mig":
                if side == "oracle":
                    r = pool.migrate(*arg)
                else:
                    c.migrate(*arg)
                    r = [(p, c.query(p, with_ids=True)[3]) for p in arg[0]]
            elif name == "reclaim":
                if side == "oracle":
                    r = [p for p, _ in pool.reclaim()]
                else:
                    moved = sorted(p for p in range(6) if _loc(c, p) == aqua.LOC_PEER)
                    c.reclaim()
                    r = moved
            elif name == "xchg":
                outs_, ins_ = arg
                if side == "oracle":
                    import copy as _copy
                    trial = _copy.deepcopy(pool)       # all-or-nothing over both lists
                    trial.swap_out(outs_)
                    r = trial.swap_in(ins_)
                    pool.__dict__.update(trial.__dict__)
                else:
                    r = c.swap_exchange(outs_, ins_, 0, 0, pieces=3)[0]
            elif name == "pstore":
                if side == "oracle":
                    r = pool.prefix_store(*arg)
                else:
                    c.prefix_store(*arg)
                    r = c.prefix_query(arg[0])
            elif name == "pload":
                r = pool.prefix_load(*arg) if side == "oracle" else c.prefix_load(*arg)[0]
            elif name == "pdrop":
                r = pool.prefix_drop(arg) if side == "oracle" else c.prefix_drop(arg)
            elif name == "relend":
                r = pool.lend(kp.LOC_PEER, arg * lay_U(pool)) if side == "oracle" else \
                    c.lend(0, FAKE * 4, arg * c.U)
        except kp.AquaError as e:
            r = ("err", e.code)
        except aqua.AquaError as e:
            r = ("err", e.code)
        res.append(r)
    return res


def _loc(c, p):
    try:
        st, loc, _ = c.query(p)
        return loc if st == aqua.SWAPPED else None
    except aqua.AquaError:
        return None


def lay_U(pool):
    return pool.lay.U


# AQUA_DRY_FUZZ_SEEDS widens this for one-off long runs (profiles/r02_dry_fuzz_long.log)
@pytest.mark.parametrize("seed", range(int(os.environ.get("AQUA_DRY_FUZZ_SEEDS", "60"))))
def test_random_op_sequences_match_oracle(seed):
    rnd = random.Random(seed)
    NB = rnd.randint(1, 24)
    lay = kp.Layout(L=1, bs=16, H=1, D=8, e=2, NB=NB)
    pool = kp.Pool(lay)
    c = aqua.Ctx(aqua.DRYRUN, 1, 16, 1, 8, 2, NB, [FAKE])
    assert c.U == lay.U
    peer = rnd.choice([0, 1, 3, 8, 16])
    host = rnd.choice([0, 2, 8])
    if peer:
        pool.lend(kp.LOC_PEER, peer * lay.U)
        c.lend(0, FAKE * 2, peer * lay.U)
    if host:
        pool.lend(kp.LOC_HOST, host * lay.U)
        c.lend(aqua.HOST, FAKE * 3, host * lay.U)
    pids = list(range(6))
    for _ in range(60):
        k = rnd.random()
        if k < 0.3:
            op = ("alloc", (rnd.choice(pids), rnd.randint(-1, 4)))
        elif k < 0.4:
            op = ("adopt", (rnd.choice(pids), [rnd.randint(-1, NB) for _ in range(rnd.randint(0, 3))]))
        elif k < 0.6:
            op = ("out", rnd.sample(pids, rnd.randint(0, 3)) + ([pids[0]] if rnd.random() < 0.05 else []))
        elif k < 0.70:
            op = ("in", rnd.sample(pids, rnd.randint(0, 3)))
        elif k < 0.75:
            sel = rnd.sample(pids, rnd.randint(0, 4))
            cut = rnd.randint(0, len(sel))
            op = ("xchg", (sel[:cut], sel[cut:]))
        elif k < 0.85:
            op = ("free", rnd.choice(pids))
        elif k < 0.93:
            op = ("mig", (rnd.sample(pids, rnd.randint(1, 2)), rnd.choice([kp.LOC_PEER, kp.LOC_HOST])))
        elif k < 0.95:
            op = ("reclaim", None)
        elif k < 0.96:
            op = ("relend", rnd.choice([1, 4, 8]))
        elif k < 0.98:
            op = ("pstore", (rnd.randint(0, 2), rnd.choice(pids), rnd.randint(-1, 3)))
        elif k < 0.995:
            op = ("pload", (rnd.randint(0, 2), rnd.choice(pids)))
        else:
            op = ("pdrop", rnd.randint(0, 2))
        a, b = _apply(pool, c, op)
        assert a == b, (seed, op, a, b)
        pool.check_invariants()
        cnt = c.counts()
        assert cnt[0] == len(pool.free)
        assert cnt[1] == (len(pool.peer.free) if pool.peer is not None else -1)
        assert cnt[2] == (len(pool.host.free) if pool.host is not None else -1)
        for f, img in pool.prefixes.items():
            assert c.prefix_query(f) == (img.location, img.slots)
        for p, pr in pool.prompts.items():
            st, loc, n, ids = c.query(p, with_ids=True)
            assert (st, loc, ids) == (pr.state, pr.location, pr.blocks if pr.state == kp.RESIDENT else pr.slots)


@pytest.mark.parametrize("slack", [0, -1, 1])
@pytest.mark.parametrize("op", ["out_peer", "out_host", "in", "mig_host", "mig_peer", "pstore", "pload", "xchg"])
def test_capacity_boundaries_match_oracle(op, slack):
    """Every capacity check at its boundary: the call needs n blocks / slots
    and exactly n + slack are free (slack 0 must succeed, -1 must fail with
    the oracle's code and change nothing, +1 succeeds).  Random sequences
    rarely land on the exact fit, so each boundary is set up on purpose."""
    n = 3
    NB = 16
    lay = kp.Layout(L=1, bs=16, H=1, D=8, e=2, NB=NB)
    pool = kp.Pool(lay)
    c = aqua.Ctx(aqua.DRYRUN, 1, 16, 1, 8, 2, NB, [FAKE])
    room = n + slack

    def both(o):
        a, b = _apply(pool, c, o)
        assert a == b, (op, slack, o, a, b)
        return a

    def lend(kind, slots):
        if kind == "peer":
            pool.lend(kp.LOC_PEER, slots * lay.U)
            c.lend(0, FAKE * 2, slots * lay.U)
        else:
            pool.lend(kp.LOC_HOST, slots * lay.U)
            c.lend(aqua.HOST, FAKE * 3, slots * lay.U)

    if op in ("out_peer", "out_host"):
        lend("peer" if op == "out_peer" else "host", room)
        both(("alloc", (1, n)))
        r = both(("out", [1]))
    elif op == "in":
        lend("peer", 8)
        both(("alloc", (1, n)))
        both(("out", [1]))
        both(("alloc", (2, NB - room)))           # leave exactly `room` free blocks
        r = both(("in", [1]))
    elif op in ("mig_host", "mig_peer"):
        src, dst = ("peer", "host") if op == "mig_host" else ("host", "peer")
        lend(src, 8)
        both(("alloc", (1, n)))
        both(("out", [1]))                       # the only arena so far: the image lands in src
        lend(dst, room)
        r = both(("mig", ([1], kp.LOC_HOST if dst == "host" else kp.LOC_PEER)))
    elif op == "pstore":
        lend("peer", room)
        both(("alloc", (1, n)))
        r = both(("pstore", (7, 1, n)))
    elif op == "pload":
        lend("peer", 8)
        both(("alloc", (1, n)))
        both(("pstore", (7, 1, n)))
        both(("alloc", (2, NB - n - room)))
        r = both(("pload", (7, 3)))
    else:                                        # exchange: the swap-outs free blocks for the resume
        lend("peer", 8)
        both(("alloc", (1, n)))
        both(("out", [1]))
        both(("alloc", (2, 2)))
        both(("alloc", (3, NB - 2 - (room - 2))))  # free blocks = room - 2; prompt 2's 2 come back
        r = both(("xchg", ([2], [1])))
    assert (r[0] == "err") == (slack < 0), (op, slack, r)
    pool.check_invariants()


def test_reclaim_order_prompts_then_prefixes_matches_oracle():
    """P:758-768 reclaim (reading in oracle.kvpool.Pool.reclaim): every image
    on the lender moves to the host -- prompts in ascending pid, then cached
    prefixes in ascending id -- into the lowest host slots in that order.
    Images interleaved on the lender (prefix, prompt, prefix, prompt) so a
    different order gives different host slots."""
    NB = 32
    lay = kp.Layout(L=1, bs=16, H=1, D=8, e=2, NB=NB)
    pool = kp.Pool(lay)
    c = aqua.Ctx(aqua.DRYRUN, 1, 16, 1, 8, 2, NB, [FAKE])
    pool.lend(kp.LOC_PEER, 16 * lay.U)
    c.lend(0, FAKE * 2, 16 * lay.U)
    pool.lend(kp.LOC_HOST, 16 * lay.U)
    c.lend(aqua.HOST, FAKE * 3, 16 * lay.U)
    ops = [("alloc", (1, 3)), ("alloc", (2, 2)), ("alloc", (3, 4)),
           ("pstore", (9, 3, 2)), ("out", [2]), ("pstore", (5, 3, 1)), ("out", [1]), ("reclaim", None)]
    for op in ops:
        a, b = _apply(pool, c, op)
        assert a == b, (op, a, b)
    for p in (1, 2):
        st, loc, n, ids = c.query(p, with_ids=True)
        assert (st, loc, ids) == (pool.prompts[p].state, pool.prompts[p].location, pool.prompts[p].slots)
    for f in (5, 9):
        assert c.prefix_query(f) == (pool.prefixes[f].location, pool.prefixes[f].slots)
    assert pool.prompts[1].slots == [0, 1, 2] and pool.prompts[2].slots == [3, 4]


def test_zero_block_image_reclaimed_without_host_matches_oracle():
    """The degenerate path the 3000-seed fuzz found in the oracle: 0-block
    images reclaimed with no host arena relocate to the host location; the
    library and the oracle agree on every later call."""
    NB = 6
    lay = kp.Layout(L=1, bs=16, H=1, D=8, e=2, NB=NB)
    pool = kp.Pool(lay)
    c = aqua.Ctx(aqua.DRYRUN, 1, 16, 1, 8, 2, NB, [FAKE])
    pool.lend(kp.LOC_PEER, 2 * lay.U)
    c.lend(0, FAKE * 2, 2 * lay.U)
    ops = [("alloc", (1, 0)), ("alloc", (2, 0)), ("alloc", (3, 2)), ("pstore", (0, 3, 0)), ("out", [1, 2]),
           ("reclaim", None), ("in", [1]), ("xchg", ([], [2])), ("out", [1]), ("free", 1), ("pload", (0, 3)),
           ("pdrop", 0), ("relend", 4), ("out", [2, 3]), ("in", [3, 2])]
    for op in ops:
        a, b = _apply(pool, c, op)
        assert a == b, (op, a, b)
        pool.check_invariants()
    assert c.counts() == (len(pool.free), len(pool.peer.free), -1)


# ------------------------------------------------------------------ CFS
def _grid():
    return [(PHASE_PREFILL, 0, 0, 0), (PHASE_PREFILL, 20, 0, 20), (PHASE_PREFILL, 40, 0, 40),
            (PHASE_DECODE, 50, 1, 50), (PHASE_DECODE, 50, 5, 54), (PHASE_DECODE, 50, 9, 58)]


@pytest.mark.parametrize("NB", [2, 4, 7, 100])
@pytest.mark.parametrize("b", [1, 3, 33, 512])
def test_partition_matches_oracle_exhaustive(NB, b):
    grid = _grid()
    for n in (1, 2, 3):
        for combo in itertools.product(range(len(grid)), repeat=n):
            s = Scheduler(NB=NB, bs=16, b=b, cap=64)
            rs = []
            for i, gi in enumerate(combo):
                ph, f, g, cx = grid[gi]
                arr = float((i * 7) % 3)
                s.add(i, arr, 50, 20)
                s.set_state(i, ph, f, g, cx)
                rs.append(ocfs.Req(id=i, arrival=arr, P=50, O=20, f=f, g=g, ctx=cx,
                                   phase=ocfs.DECODE if ph == PHASE_DECODE else ocfs.PREFILL))
            D, PF = s.partition()
            oD, oPF = ocfs.plan(rs, b, NB, 16)
            assert (D, [tuple(x) for x in PF]) == (oD, [tuple(x) for x in oPF]), combo
            s.close()


def test_partition_random_states_match_oracle():
    rnd = random.Random(7)
    for trial in range(400):
        n = rnd.randint(1, 12)
        NB = rnd.randint(1, 60)
        b = rnd.choice([1, 8, 64, 512])
        bs = rnd.choice([1, 4, 16])
        s = Scheduler(NB=NB, bs=bs, b=b, cap=64)
        rs = []
        for i in range(n):
            P = rnd.randint(1, 300)
            O = rnd.randint(1, 50)
            if rnd.random() < 0.5:
                f = rnd.randint(0, P - 1)
                ph, g, cx = PHASE_PREFILL, 0, f
            else:
                f, g = P, rnd.randint(1, O)
                ph, cx = PHASE_DECODE, P + g - 1
            arr = float(rnd.randint(0, 5))
            s.add(i, arr, P, O)
            s.set_state(i, ph, f, g, cx)
            rs.append(ocfs.Req(id=i, arrival=arr, P=P, O=O, f=f, g=g, ctx=cx,
                               phase=ocfs.DECODE if ph == PHASE_DECODE else ocfs.PREFILL))
        D, PF = s.partition()
        oD, oPF = ocfs.plan(rs, b, NB, bs)
        assert (D, [tuple(x) for x in PF]) == (oD, [tuple(x) for x in oPF]), trial
        s.close()


def _product_log(trace, NB, lender_slots, host_slots, policy=POLICY_CFS, k=8, b=512, bs=16):
    c = aqua.Ctx(aqua.DRYRUN, 1, bs, 1, 8, 2, NB, [FAKE])
    if lender_slots:
        c.lend(0, FAKE * 2, lender_slots * c.U)
    if host_slots:
        c.lend(aqua.HOST, FAKE * 3, host_slots * c.U)
    s = Scheduler(NB=NB, bs=bs, b=b, k=k, policy=policy)
    log, st = run_trace(trace, c, s)
    return log, st


@pytest.mark.parametrize("policy", ["cfs", "fcfs"])
def test_more_decoding_prompts_than_the_batch_budget(policy):
    """b = 4 tokens per iteration and 9 prompts decoding at once (restarted
    prompts, R19; ample memory): FCFS decodes the 4 earliest arrivals per
    iteration (SPEC fcfs_step S:297-305), CFS the 4 least served.  The call
    logs (plans, iterations) equal the oracle's."""
    tr = [(i, 0.001 * i, 8, 12) for i in range(9)]
    warm = [i for i, *_ in tr]                   # R19: all nine arrive decoding, images paged out
    o = osim.run(tr, osim.SimConfig(NB=64, bs=16, b=4, k=3, policy=policy, lender_slots=0, host_slots=64,
                                    max_iters=40), warm=warm)
    c = aqua.Ctx(aqua.DRYRUN, 1, 16, 1, 8, 2, 64, [FAKE])
    c.lend(aqua.HOST, FAKE * 3, 64 * c.U)
    s = Scheduler(NB=64, bs=16, b=4, k=3, policy=POLICY_CFS if policy == "cfs" else POLICY_FCFS)
    log, _ = run_trace(tr, c, s, warm=warm, max_iters=40)
    assert log == o.log
    assert max(len(e[2]) for e in o.log if e[0] == "iter") == 4


@pytest.mark.parametrize("policy", ["cfs", "fcfs"])
@pytest.mark.parametrize("k", [1, 8])
def test_small_trace_call_log_matches_oracle(policy, k):
    tr = burst_trace(seed=3, burst_s=8.0, tail_s=3.0, prompt=(300, 0.8, 1, 900), output=(40, 0.7, 1, 200))
    NB = 120
    o = osim.run(tr, osim.SimConfig(NB=NB, k=k, policy=policy, lender_slots=200, host_slots=400))
    log, st = _product_log(tr, NB, 200, 400, policy=POLICY_CFS if policy == "cfs" else POLICY_FCFS, k=k)
    assert st["iters"] == o.iters
    assert len(log) == len(o.log)
    for a, b in zip(log, o.log):
        assert a == b
    if policy == "cfs":
        assert o.blocks_out > 0 and st["blocks_out"] == o.blocks_out


def test_lender_overflow_falls_back_to_host_in_trace():
    tr = burst_trace(seed=5, burst_s=8.0, tail_s=3.0, prompt=(300, 0.8, 1, 900), output=(40, 0.7, 1, 200))
    o = osim.run(tr, osim.SimConfig(NB=100, lender_slots=30, host_slots=1000))
    log, _ = _product_log(tr, 100, 30, 1000)
    assert log == o.log
    locs = {loc for e in o.log if e[0] == "swap_out" for loc, _ in e[2]}
    assert locs == {kp.LOC_PEER, kp.LOC_HOST}


def test_full_c3_trace_call_log_matches_oracle():
    """BASELINE configs[2] at full size, metadata mode (seed 1): the native
    scheduler + libaqua bookkeeping reproduce the oracle's call log."""
    tr = burst_trace(seed=1)
    NB = 4152                       # scripts/c3_nb.py (oracle FCFS pre-burst peak x 1.2)
    o = osim.run(tr, osim.SimConfig(NB=NB, lender_slots=32768, host_slots=32768))
    log, st = _product_log(tr, NB, 32768, 32768)
    assert st["iters"] == o.iters and st["blocks_out"] == o.blocks_out
    assert log == o.log


@pytest.mark.parametrize("n,m,k", [(n, m, k) for n in (1, 3, 5, 6) for m in range(1, n + 1) for k in (1, 2, 3)])
def test_round_robin_call_log_matches_oracle(n, m, k):
    """C-9 instances (decode-only, bs=64, NB=m, ids in reverse arrival order;
    the oracle side is pinned to the deque-rotation model in
    test_oracle_cfs.py): the native scheduler + libaqua give the same log."""
    order = [100 + n - 1 - j for j in range(n)]
    tr = [(pid, -100.0 + j, 8, 10 ** 6) for j, pid in enumerate(order)]
    o = osim.run(tr, osim.SimConfig(NB=m, bs=64, b=512, k=k, host_slots=64, max_iters=30), warm=order)
    c = aqua.Ctx(aqua.DRYRUN, 1, 64, 1, 8, 2, m, [FAKE])
    c.lend(aqua.HOST, FAKE * 3, 64 * c.U)
    s = Scheduler(NB=m, bs=64, b=512, k=k)
    log, st = run_trace(tr, c, s, warm=order, max_iters=30)
    assert log == o.log
    assert st["blocks_out"] == o.blocks_out and st["blocks_in"] == o.blocks_in


def test_scheduler_failed_calls_change_nothing():
    """aqua_cfs_next / aqua_cfs_commit with a too-small output capacity fail
    with AQUA_E_INVAL and leave the scheduler as it was: a retry with room
    gives exactly what an untouched twin gives (all-or-nothing, like the
    paging calls)."""
    def mk():
        s = Scheduler(NB=2, bs=64, b=512, k=1, cap=64)
        for j in range(4):
            s.add(10 + j, float(j), 8, 3)
            s.set_state(10 + j, PHASE_DECODE, 8, 1, 8)      # restart: image swapped out
        return s
    a, b = mk(), mk()
    for it in range(12):
        if a.stats()[0] == 0:
            break
        a.cap = 1
        with pytest.raises(aqua.AquaError) as ei:
            a.next()
        assert ei.value.code == aqua.E_INVAL
        a.cap = 64
        ra, rb = a.next(), b.next()
        assert ra == rb, it
        fb = b.commit()
        if fb[0]:
            a.cap = len(fb[0]) - 1
            with pytest.raises(aqua.AquaError):
                a.commit()
            a.cap = 64
        assert a.commit() == fb
        assert a.stats() == b.stats() and a.vclock() == b.vclock()
    assert a.stats()[0] == 0


def test_reoffer_with_unequal_images_matches_oracle():
    """R22 through the product: the driver's re-offer moves host images back
    in ascending pid while they fit and stops at the first that does not --
    a scenario (unequal image sizes, 12 re-offered slots) where skipping
    ahead would move a different set.  Call log equal to the oracle's."""
    Ps = (40, 200, 40, 40, 120, 40, 40, 40)
    tr = [(i, 0.01 * i, Ps[i], 300) for i in range(8)]
    NB, lender, host = 40, 400, 2000
    o = osim.run(tr, osim.SimConfig(NB=NB, b=64, lender_slots=lender, host_slots=host, elastic=(2.0, 3.0),
                                    relend_slots=12))
    c = aqua.Ctx(aqua.DRYRUN, 1, 16, 1, 8, 2, NB, [FAKE])
    c.lend(0, FAKE * 2, lender * c.U)
    c.lend(aqua.HOST, FAKE * 3, host * c.U)
    s = Scheduler(NB=NB, bs=16, b=64, k=8)
    log, _ = run_trace(tr, c, s, elastic={"t_reclaim": 2.0, "t_relend": 3.0, "relend": (0, FAKE * 5, 12 * c.U)})
    assert any(e[0] == "migrate" for e in o.log)
    assert log == o.log


@pytest.mark.parametrize("window", [(4.0, 9.0), (2.0, 30.0), (6.0, 6.5)])
def test_elastic_trace_call_log_matches_oracle(window):
    """NEXT-1 end to end in metadata mode: lender reclaim -> images to DRAM,
    FCFS fallback, re-offer -> images back, CFS again; the
    product's call log equals the oracle's."""
    tr = burst_trace(seed=3, burst_s=8.0, tail_s=3.0, prompt=(300, 0.8, 1, 900), output=(40, 0.7, 1, 200))
    NB, lender, host = 120, 400, 2000
    o = osim.run(tr, osim.SimConfig(NB=NB, lender_slots=lender, host_slots=host, elastic=window,
                                    relend_slots=lender))
    c = aqua.Ctx(aqua.DRYRUN, 1, 16, 1, 8, 2, NB, [FAKE])
    c.lend(0, FAKE * 2, lender * c.U)
    c.lend(aqua.HOST, FAKE * 3, host * c.U)
    s = Scheduler(NB=NB, bs=16, b=512, k=8)
    log, st = run_trace(tr, c, s, elastic={"t_reclaim": window[0], "t_relend": window[1],
                                          "relend": (0, FAKE * 5, lender * c.U)})
    kinds = [e[0] for e in o.log]
    assert "reclaim" in kinds and ("relend" in kinds) == (window[1] < o.vclock)
    assert log == o.log
    # while the images sit in DRAM no swap_out goes to the (absent) lender
    fb = False
    for e in o.log:
        if e[0] == "policy":
            fb = e[2] == "fcfs"
        if fb and e[0] == "swap_out":
            assert all(loc == kp.LOC_HOST for loc, _ in e[2])
        if fb:
            assert e[0] != "plan"


def test_fallback_overflow_preemption_matches_oracle():
    """FCFS fallback inheriting more residents than their projections allow:
    growth overflows and the latest-arrived resident is paged out (R18);
    swapped prompts are paged in when admitted."""
    tr = [(i, 0.01 * i, 40, 300) for i in range(8)]
    NB = 40
    o = osim.run(tr, osim.SimConfig(NB=NB, b=64, lender_slots=400, host_slots=2000, elastic=(0.5, 1e9),
                                    relend_slots=400))
    fb = [e for e in o.log if e[0] in ("swap_out", "swap_in")
          and o.log.index(e) > [x[0] for x in o.log].index("policy")]
    assert any(e[0] == "swap_out" for e in fb) and any(e[0] == "swap_in" for e in fb)
    c = aqua.Ctx(aqua.DRYRUN, 1, 16, 1, 8, 2, NB, [FAKE])
    c.lend(0, FAKE * 2, 400 * c.U)
    c.lend(aqua.HOST, FAKE * 3, 2000 * c.U)
    s = Scheduler(NB=NB, bs=16, b=64, k=8)
    log, _ = run_trace(tr, c, s, elastic={"t_reclaim": 0.5, "t_relend": 1e9, "relend": (0, FAKE * 5, 400 * c.U)})
    assert log == o.log


def test_layered_calls_same_bookkeeping_dryrun():
    c = dry_ctx(L=5, NB=20)
    c.lend(0, FAKE * 2, 20 * c.U)
    c.alloc_blocks(1, 4)
    t = c.swap_out_layers([1], 2)
    assert len(t) == 3 and len(set(t)) == 1
    assert c.query(1, with_ids=True)[3] == [0, 1, 2, 3]
    new, t = c.swap_in_layers([1], 5)
    assert new == [[0, 1, 2, 3]] and len(t) == 1
    with pytest.raises(aqua.AquaError):
        c.swap_out_layers([1], 0)


def test_exchange_driver_call_log_matches_oracle():
    """Reschedules issued as aqua_swap_exchange keep the oracle's call log."""
    tr = burst_trace(seed=3, burst_s=8.0, tail_s=3.0, prompt=(300, 0.8, 1, 900), output=(40, 0.7, 1, 200))
    NB = 120
    o = osim.run(tr, osim.SimConfig(NB=NB, lender_slots=200, host_slots=400))
    c = aqua.Ctx(aqua.DRYRUN, 1, 16, 1, 8, 2, NB, [FAKE])
    c.lend(0, FAKE * 2, 200 * c.U)
    c.lend(aqua.HOST, FAKE * 3, 400 * c.U)
    log, st = run_trace(tr, c, Scheduler(NB=NB, bs=16), exchange_stream=0)
    assert log == o.log


@pytest.mark.parametrize("exchange", [False, True])
def test_native_trace_runner_matches_oracle(exchange):
    """aqua_trace_run (the engine loop in C++) reproduces the oracle's call
    log on the full C3 trace (dry-run ctx: bookkeeping only)."""
    from paper_2407_21255_b200.cfs import run_trace_native
    tr = burst_trace(seed=1)
    NB = 4152
    o = osim.run(tr, osim.SimConfig(NB=NB, lender_slots=32768, host_slots=32768))
    c = aqua.Ctx(aqua.DRYRUN, 1, 16, 1, 8, 2, NB, [FAKE])
    c.lend(0, FAKE * 2, 32768 * c.U)
    c.lend(aqua.HOST, FAKE * 3, 32768 * c.U)
    log, st = run_trace_native(tr, c, Scheduler(NB=NB, bs=16), swap_stream2=1 if exchange else 0)
    assert st["iters"] == o.iters and st["blocks_out"] == o.blocks_out
    assert log == o.log


# AQUA_TRACE_FUZZ_SEEDS widens this for one-off long runs (profiles/r02_trace_fuzz_long.log)
# seed 2455: an FCFS fallback that overflows by two residents (R18: one call, latest arrival first)
@pytest.mark.parametrize("seed", sorted(set(range(int(os.environ.get("AQUA_TRACE_FUZZ_SEEDS", "12")))) | {2455}))
def test_random_trace_call_logs_match_oracle(seed):
    """Random bursty traces and engine settings -- pool size, block size,
    time-slice k, budget b, CFS or FCFS, lender and host capacities down to
    none (so preemptions overflow to the host or stall), occasionally the
    elastic reclaim / re-offer -- through the Python driver and the native
    C++ trace runner, both over the native scheduler and the dry-run library:
    the whole call log must equal the oracle's sim.run log."""
    from paper_2407_21255_b200.cfs import run_trace_native
    rnd = random.Random(seed)
    bs = rnd.choice([4, 16])
    maxP, maxO = rnd.choice([(200, 60), (600, 120), (900, 200)])
    tr = burst_trace(seed=100 + seed, lam0=rnd.choice([1.5, 2.5, 6.0]), n_pre=rnd.randint(1, 25),
                     burst_mult=rnd.choice([1.0, 2.0, 4.0]), burst_s=rnd.uniform(1.0, 8.0), tail_s=rnd.uniform(0.0, 3.0),
                     prompt=(maxP // 3, 0.8, 1, maxP), output=(maxO // 4, 0.7, 1, maxO))
    need = -(-(maxP + maxO) // bs)                     # blocks of the longest request
    NB = need + rnd.randint(1, 4 * need)
    k = rnd.choice([1, 2, 3, 8])
    b = rnd.choice([64, 512])
    policy = rnd.choice(["cfs", "cfs", "fcfs"])
    # swap space never runs out (the paper's DRAM fallback is 1.5 TB; neither side defines a
    # preemption with nowhere to go): the lender may be small or absent, the host then holds everything
    total = len(tr) * need
    lender = rnd.choice([0, NB // 4, NB, total])
    host = total if lender < total else rnd.choice([0, total])
    elastic = None
    if lender and host and rnd.random() < 0.25:
        elastic = (rnd.uniform(0.2, 4.0), rnd.choice([rnd.uniform(4.0, 9.0), 1e9]))
    cfg = osim.SimConfig(NB=NB, bs=bs, b=b, k=k, policy=policy, lender_slots=lender, host_slots=host,
                         elastic=elastic, relend_slots=lender if elastic else 0)
    o = osim.run(tr, cfg)
    pol = POLICY_CFS if policy == "cfs" else POLICY_FCFS

    def ctx():
        c = aqua.Ctx(aqua.DRYRUN, 1, bs, 1, 8, 2, NB, [FAKE])
        if lender:
            c.lend(0, FAKE * 2, lender * c.U)
        if host:
            c.lend(aqua.HOST, FAKE * 3, host * c.U)
        return c

    kw = {}
    if elastic:
        c0 = ctx()
        kw["elastic"] = {"t_reclaim": elastic[0], "t_relend": elastic[1], "relend": (0, FAKE * 5, lender * c0.U)}
        kw["policy_after_relend"] = pol
        c0.close()
    if rnd.random() < 0.3:                             # reschedules issued as aqua_swap_exchange
        kw["exchange_stream"] = 0
        kw["exchange_pieces"] = rnd.choice([1, 3, 16])
    log, st = run_trace(tr, ctx(), Scheduler(NB=NB, bs=bs, b=b, k=k, policy=pol), **kw)
    assert st["iters"] == o.iters, (seed, cfg, kw)
    assert log == o.log, (seed, cfg, kw)
    if not elastic:                                    # the native runner has no elastic hooks
        nlog, nst = run_trace_native(tr, ctx(), Scheduler(NB=NB, bs=bs, b=b, k=k, policy=pol),
                                     swap_stream2=rnd.choice([0, 1]))
        assert nlog == o.log and nst["iters"] == o.iters, (seed, cfg)


def test_create_validates_layout():
    """aqua_create rejects layouts the kernels cannot move exactly (S or a
    stride not a multiple of 16, overlapping chunks, misaligned bases)."""
    ok = aqua.Ctx(aqua.DRYRUN, 2, 16, 2, 64, 2, 8, [FAKE, FAKE + (1 << 30)])
    ok.close()
    bad = [
        dict(L=1, bs=1, H=1, D=4, e=2, NB=4, ptrs=[FAKE]),                                   # S = 8 bytes
        dict(L=1, bs=16, H=1, D=8, e=2, NB=4, ptrs=[FAKE + 8]),                              # misaligned base
        dict(L=1, bs=16, H=1, D=8, e=2, NB=4, ptrs=[FAKE], kv=16, blk=256),                  # K/V planes overlap
        dict(L=1, bs=16, H=1, D=8, e=2, NB=4, ptrs=[FAKE], kv=0, blk=128),                   # blocks overlap
        dict(L=0, bs=16, H=1, D=8, e=2, NB=4, ptrs=[]),
        dict(L=1, bs=16, H=1, D=8, e=2, NB=0, ptrs=[FAKE]),
    ]
    for b in bad:
        with pytest.raises(aqua.AquaError) as e:
            aqua.Ctx(aqua.DRYRUN, b["L"], b["bs"], b["H"], b["D"], b["e"], b["NB"], b["ptrs"],
                     b.get("kv", 0), b.get("blk", 0))
        assert e.value.code == aqua.E_INVAL
    c = aqua.Ctx(aqua.DRYRUN, 1, 16, 1, 8, 2, 4, [FAKE])
    for opt, val in ((aqua.OPT_KERNEL, 99), (aqua.OPT_TMA_PIECE, 17), (aqua.OPT_TMA_STAGES, 1),
                     (aqua.OPT_MAX_CTAS, -1), (aqua.OPT_TIMING, 2), (aqua.OPT_LDST_VARIANT, 4),
                     (aqua.OPT_TMA_VARIANT, 4), (aqua.OPT_INLINE_MAX, 4065), (aqua.OPT_INLINE_MAX, -1),
                     (aqua.OPT_TMA_STATIC_PCT, 101), (aqua.OPT_RATE_GBPS, -1), (aqua.OPT_PEER_CTAS, -1),
                     (aqua.OPT_PEER_TEST, 3),
                     # round 1's experiments, retired in round 2
                     (aqua.OPT_LDST_VARIANT, 0), (aqua.OPT_LDST_VARIANT, 1), (aqua.OPT_TMA_VARIANT, 1),
                     (aqua.OPT_TMA_VARIANT, 2), (aqua.OPT_TMA_VARIANT, 4), (aqua.OPT_TMA_SCHED, -3), (aqua.OPT_TMA_STATIC_PCT, 60),
                     (77, 0)):
        with pytest.raises(aqua.AquaError):
            c.set_option(opt, val)
    assert c.get_option(aqua.OPT_INLINE_MAX) == 4064              # the 32,764-byte parameter limit
    assert c.get_option(aqua.OPT_TMA_SCHED) == aqua.TMA_SCHED_AUTO
    with pytest.raises(aqua.AquaError) as e:
        c.last_launch()                                          # a dry-run context never launches
    assert e.value.code == aqua.E_STATE
    c.set_option(aqua.OPT_TMA_SCHED, 8)
    c.set_option(aqua.OPT_TMA_SCHED, aqua.TMA_SCHED_AUTO)
    assert c.get_option(aqua.OPT_PEER_CTAS) == 32
    c.set_option(aqua.OPT_INLINE_MAX, 0)
    assert c.get_option(aqua.OPT_INLINE_MAX) == 0
    with pytest.raises(aqua.AquaError) as e:
        c.lend(0, FAKE + 8, 4096)                                                             # misaligned arena
    assert e.value.code == aqua.E_INVAL
    c.lend(0, FAKE * 2, 10 * c.U)
    with pytest.raises(aqua.AquaError) as e:
        c.lend(0, FAKE * 3, 10 * c.U)                                                         # one GPU lender
    assert e.value.code == aqua.E_INVAL
