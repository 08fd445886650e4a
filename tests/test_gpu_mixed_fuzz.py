"""GPU parity on random MIXED operation sequences (-m gpu): every library
call that moves bytes -- alloc, adopt, swap_out, swap_in, exchange, free,
migrate, reclaim, re-lend, prefix store / load / drop, layer-wise swaps --
in random order and with random arguments (many of them invalid), on the
sm_100a kernels through the C ABI against the CPU oracle in bytes mode.
After every call the pool, the lender arena and the host arena are compared
whole-buffer; a failing call must fail with the oracle's code and change
nothing (all-or-nothing).  The dry-run fuzz (test_dryrun_parity.py)
checks the same op mix on bookkeeping alone at 50,000 seeds; this one checks
the bytes.  AQUA_FUZZ_SEEDS / AQUA_FUZZ_OPS widen it for one-off runs."""
import copy
import os
import random

import numpy as np
import pytest
import torch

from oracle import kvpool as kp
from paper_2407_21255_b200 import aqua
from workloads import kv_random_bytes

from gpu_util import Rig

pytestmark = pytest.mark.gpu

SEEDS = list(range(int(os.environ.get("AQUA_FUZZ_SEEDS", "3"))))
NOPS = int(os.environ.get("AQUA_FUZZ_OPS", "40"))
SHAPES = {"c4_8KiB": (3, 16, 2, 128), "s512": (3, 16, 1, 16), "ragged_10KiB": (2, 16, 5, 64)}
ENGINES = {"auto": (aqua.KERNEL_AUTO, 0, 2), "tma": (aqua.KERNEL_TMA, 0, 2), "hybrid": (aqua.KERNEL_TMA, 3, 2),
           "ldst": (aqua.KERNEL_LDST, 0, 2), "small": (aqua.KERNEL_LDST, 0, 3), "ce_host": (aqua.KERNEL_CE_HOST, 0, 2)}
LOCS = {kp.LOC_PEER: aqua.LOC_PEER, kp.LOC_HOST: aqua.LOC_HOST}


def _gen(rnd, pids, L, o):
    """One random op.  Four times in five the pids come from the state the op
    needs (resident for out / prefix store, swapped for in / migrate), so that
    most calls succeed; otherwise from all pids, which exercises the errors."""
    res = [p for p, pr in o.prompts.items() if pr.state == kp.RESIDENT]
    swp = [p for p, pr in o.prompts.items() if pr.state == kp.SWAPPED]
    fids = list(o.prefixes)

    def pick(valid, k):
        pool = valid if valid and rnd.random() < 0.8 else pids
        return rnd.sample(pool, min(len(pool), rnd.randint(1, k)))

    k = rnd.random()
    if k < 0.20:
        return ("alloc", (rnd.choice(pids), rnd.randint(0, 4)))
    if k < 0.24:
        return ("adopt", (rnd.choice(pids), [rnd.randint(-1, 30) for _ in range(rnd.randint(0, 3))]))
    if k < 0.42:
        return ("out", pick(res, 3))
    if k < 0.58:
        return ("in", pick(swp, 3))
    if k < 0.64:
        a, b = pick(res, 2), pick(swp, 2)
        return ("xchg", ([p for p in a if p not in b], b, rnd.choice([1, 3])))
    if k < 0.72:
        return ("free", rnd.choice(pids))
    if k < 0.78:
        sel = pick(swp, 2)
        here = {o.prompts[p].location for p in sel if p in o.prompts and o.prompts[p].state == kp.SWAPPED}
        dst = ({kp.LOC_PEER, kp.LOC_HOST} - here).pop() if len(here) == 1 and rnd.random() < 0.8 else \
            rnd.choice([kp.LOC_PEER, kp.LOC_HOST])
        return ("mig", (sel, dst))
    if k < 0.81:
        return ("reclaim", None)
    if k < 0.84:
        return ("relend", rnd.choice([2, 6, 12]))
    if k < 0.89:
        return ("pstore", (rnd.randint(0, 2), pick(res, 1)[0], rnd.randint(-1, 3)))
    if k < 0.93:
        return ("pload", (rnd.choice(fids) if fids and rnd.random() < 0.8 else rnd.randint(0, 2),
                          rnd.choice(res) if res and rnd.random() < 0.8 else rnd.choice(pids + [7, 8])))
    if k < 0.95:
        return ("pdrop", rnd.choice(fids) if fids and rnd.random() < 0.8 else rnd.randint(0, 2))
    if k < 0.975:
        return ("out_layers", (pick(res, 2), rnd.randint(1, L)))
    return ("in_layers", (pick(swp, 2), rnd.randint(1, L)))


def _oracle(o, op):
    name, arg = op
    if name == "alloc":
        return o.alloc_blocks(*arg)
    if name == "adopt":
        return o.adopt_blocks(*arg)
    if name in ("out", "out_layers"):
        return [(loc, s) for _, loc, s in o.swap_out(arg if name == "out" else arg[0])]
    if name in ("in", "in_layers"):
        return o.swap_in(arg if name == "in" else arg[0])
    if name == "xchg":
        trial = copy.deepcopy(o)                 # all-or-nothing over both lists
        trial.swap_out(arg[0])
        r = trial.swap_in(arg[1])
        o.__dict__.update(trial.__dict__)
        return r
    if name == "free":
        return o.free_prompt(arg)
    if name == "mig":
        return o.migrate(*arg)
    if name == "reclaim":
        return [p for p, _ in o.reclaim()]
    if name == "pstore":
        return o.prefix_store(*arg)
    if name == "pload":
        return o.prefix_load(*arg)
    if name == "pdrop":
        return o.prefix_drop(arg)
    raise AssertionError(name)


def _lib(rig, op, moved_before):
    c = rig.ctx
    name, arg = op
    if name == "alloc":
        return c.alloc_blocks(*arg)
    if name == "adopt":
        return c.adopt_blocks(*arg)
    if name in ("out", "out_layers"):
        pids = arg if name == "out" else arg[0]
        if name == "out":
            c.swap_out(pids)
        else:
            c.swap_out_layers(pids, arg[1])
        return [(c.query(p)[1], c.query(p, with_ids=True)[3]) for p in pids]
    if name == "in":
        return c.swap_in(arg, cap=4096)[0]
    if name == "in_layers":
        return c.swap_in_layers(arg[0], arg[1])[0]
    if name == "xchg":
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        return c.swap_exchange(arg[0], arg[1], s1.cuda_stream, s2.cuda_stream, pieces=arg[2])[0]
    if name == "free":
        return c.free(arg)
    if name == "mig":
        c.migrate(arg[0], LOCS[arg[1]])
        return [(p, c.query(p, with_ids=True)[3]) for p in arg[0]]
    if name == "reclaim":
        c.reclaim()
        return moved_before
    if name == "pstore":
        c.prefix_store(*arg)
        loc, slots = c.prefix_query(arg[0])
        return ({aqua.LOC_PEER: kp.LOC_PEER, aqua.LOC_HOST: kp.LOC_HOST}[loc], slots)
    if name == "pload":
        return c.prefix_load(*arg)[0]
    if name == "pdrop":
        return c.prefix_drop(arg)
    raise AssertionError(name)


def _peer_pids(c, pids):
    out = []
    for p in pids:
        try:
            st, loc, _ = c.query(p)
        except aqua.AquaError:
            continue
        if st == aqua.SWAPPED and loc == aqua.LOC_PEER:
            out.append(p)
    return sorted(out)


def _counts_equal(rig):
    o = rig.opool
    assert rig.ctx.counts() == (len(o.free), len(o.peer.free) if o.peer is not None else -1,
                                len(o.host.free) if o.host is not None else -1)


@pytest.mark.parametrize("shape", list(SHAPES))
@pytest.mark.parametrize("engine", list(ENGINES))
@pytest.mark.parametrize("seed", SEEDS)
def test_random_mixed_sequences_bytes(shape, engine, seed):
    L, bs, H, D = SHAPES[shape]
    rnd = random.Random(1000 * seed + 17 * len(shape) + len(engine))
    rig = Rig(L=L, bs=bs, H=H, D=D, NB=30, lender_slots=rnd.choice([0, 6, 12]), host_slots=rnd.choice([0, 8, 16]),
              seed=seed)
    c, o = rig.ctx, rig.opool
    kern, tv, lv = ENGINES[engine]
    c.set_option(aqua.OPT_KERNEL, kern)
    c.set_option(aqua.OPT_TMA_VARIANT, tv)
    c.set_option(aqua.OPT_LDST_VARIANT, lv)
    if shape == "ragged_10KiB" and engine in ("tma", "hybrid"):
        c.set_option(aqua.OPT_TMA_PIECE, 4096)
    keep = []                                   # arenas the library may still read until their tickets pass
    pids = list(range(6))
    U = rig.lay.U
    for i in range(NOPS):
        op = _gen(rnd, pids, L, o)
        if op[0] == "relend":
            n = op[1]
            g = kv_random_bytes(n * U, seed=5000 + 31 * seed + i)
            t = torch.from_numpy(g.copy()).cuda()
            try:
                o.lend(kp.LOC_PEER, n * U, g.copy())
                code_o = None
            except kp.AquaError as e:
                code_o = e.code
            try:
                c.lend(0, t.data_ptr(), n * U)
                code_c = None
            except aqua.AquaError as e:
                code_c = e.code
            assert code_o == code_c, (i, op, code_o, code_c)
            if code_c is None:
                rig.peer = t
                keep.append(t)
        else:
            moved = _peer_pids(c, range(10)) if op[0] == "reclaim" else None   # pload may create pids 7, 8
            if op[0] == "reclaim" and o.peer is not None and moved != sorted(
                    p for p, pr in o.prompts.items() if pr.state == kp.SWAPPED and pr.location == kp.LOC_PEER):
                raise AssertionError((i, "lender images differ before reclaim"))
            snap = copy.deepcopy(o)
            try:
                want = _oracle(o, op)
                code_o = None
            except kp.AquaError as e:
                want, code_o = None, e.code
                o.__dict__.update(snap.__dict__)
            try:
                got = _lib(rig, op, moved)
                code_c = None
            except aqua.AquaError as e:
                got, code_c = None, e.code
            assert code_o == code_c, (i, op, code_o, code_c)
            if code_c is None:
                assert got == want, (i, op, got, want)
            if op[0] == "reclaim" and code_c is None and o.peer is None and rig.peer is not None:
                keep.append(rig.peer)
                rig.peer = None
        rig.assert_bytes_equal(f"op {i} {op}")
        _counts_equal(rig)
        o.check_invariants()
        for p, pr in o.prompts.items():
            st, loc, n, ids = c.query(p, with_ids=True)
            assert (st, ids) == (pr.state, pr.blocks if pr.state == kp.RESIDENT else pr.slots), (i, p)
    torch.cuda.synchronize()
