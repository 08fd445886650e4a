"""Pins for oracle/kvpool.py against things other than itself.

* the C1 golden script (tests/golden/c1_script.json, hand-derived ids);
* byte results recomputed through the *meaning* of the layout (an
  [2][NB][S] reshape of each layer, [nslots][L][2][S] of the arena) rather
  than the oracle's offset arithmetic;
* the L=1, NB=1 special case (swap == memcpy of the whole layer);
* SPEC's allocation examples re-expressed in slots;
* exhaustive brute force of short op sequences against a tiny array-scan
  model of the allocator, with all-or-nothing checked on every failure.
"""
import copy
import itertools
import json
import os

import numpy as np
import pytest

from oracle import kvpool as kp
from workloads import kv_random_bytes

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def make_pool(L=2, H=2, D=64, e=2, bs=16, NB=40, seed=0, **kw):
    lay = kp.Layout(L=L, bs=bs, H=H, D=D, e=e, NB=NB, **kw)
    layers = [kv_random_bytes(lay.layer_bytes, seed=seed + l).copy() for l in range(L)]
    return kp.Pool(lay, layers)


def planes(pool):
    """[L][2][NB][S] view via the flash layout's meaning (R1), not offsets."""
    lay = pool.lay
    return np.stack([a[:2 * lay.NB * lay.S].reshape(2, lay.NB, lay.S) for a in pool.layers])


def run_c1(lender_slots, host_slots=0):
    g = json.load(open(os.path.join(GOLD, "c1_script.json")))
    lay = g["layout"]
    pool = make_pool(**lay)
    U = pool.lay.U
    peer = kv_random_bytes(lender_slots * U, seed=100).copy()
    pool.lend(kp.LOC_PEER, lender_slots * U, peer)
    host = None
    if host_slots:
        host = kv_random_bytes(host_slots * U, seed=101).copy()
        pool.lend(kp.LOC_HOST, host_slots * U, host)
    for p in range(g["prompts"]):
        assert pool.alloc_blocks(p, g["blocks_per_prompt"]) == g["initial_ids"][str(p)]
    return g, pool, peer, host


@pytest.mark.parametrize("variant", ["lender12", "lender8"])
def test_c1_golden_script(variant):
    g0 = json.load(open(os.path.join(GOLD, "c1_script.json")))
    v = g0[variant]
    g, pool, peer, host = run_c1(v["lender_slots"], v.get("host_slots", 0))
    before = planes(pool).copy()
    peer0 = peer.copy()
    res = pool.swap_out(g["swap_out"])
    pool.check_invariants()
    for pid, loc, slots in res:
        want_loc, want_slots = v["placement"][str(pid)]
        assert loc == {"peer": kp.LOC_PEER, "host": kp.LOC_HOST}[want_loc]
        assert slots == want_slots
    # pool untouched by swap_out (I2)
    assert np.array_equal(planes(pool), before)
    # image formula (I5) through the [slot][L][2][S] meaning of the arena
    for pid, loc, slots in res:
        ar = (peer if loc == kp.LOC_PEER else host).reshape(-1, pool.lay.L, 2, pool.lay.S)
        for j, s in enumerate(slots):
            b = g["initial_ids"][str(pid)][j]
            assert np.array_equal(ar[s], before[:, :, b, :])
    # untouched slots keep their garbage (I2)
    used_peer = {s for pid, loc, sl in res if loc == kp.LOC_PEER for s in sl}
    arp, arp0 = peer.reshape(-1, pool.lay.U), peer0.reshape(-1, pool.lay.U)
    for s in range(v["lender_slots"]):
        if s not in used_peer:
            assert np.array_equal(arp[s], arp0[s])
    assert pool.alloc_blocks(g["filler"]["pid"], g["filler"]["n"]) == g["filler"]["expected_ids"]
    mid = planes(pool).copy()
    new = pool.swap_in(g["swap_in"])
    pool.check_invariants()
    for pid, ids in zip(g["swap_in"], new):
        assert ids == g["expected_swap_in_ids"][str(pid)]
    after = planes(pool)
    # restore (I1) + non-interference (I2): only the new blocks changed
    expect = mid.copy()
    for pid, ids in zip(g["swap_in"], new):
        for j, b in enumerate(ids):
            expect[:, :, b, :] = before[:, :, g["initial_ids"][str(pid)][j], :]
    assert np.array_equal(after, expect)
    pool.free_prompt(g["filler"]["pid"])
    pool.check_invariants()
    assert len(pool.free) == 40 - 8 * 4


def test_single_block_is_memcpy():
    """L=1, NB=1: the swap image of the only block is the layer verbatim."""
    pool = make_pool(L=1, NB=1, H=1, D=8, bs=16)
    lay = pool.lay
    arena = np.zeros(lay.U, np.uint8)
    pool.lend(kp.LOC_PEER, lay.U, arena)
    pool.alloc_blocks(7, 1)
    layer = pool.layers[0].copy()
    pool.swap_out([7])
    assert np.array_equal(arena, layer[:2 * lay.S])
    pool.layers[0][:] = 0
    assert pool.swap_in([7]) == [[0]]
    assert np.array_equal(pool.layers[0], layer)


def test_block_major_layout_strides():
    """Generic strides: vLLM's [NB][2][bs][H][D] layout (P_kv = S,
    P_b = 2S) must give the same images as the plain meaning of that
    layout (a [NB][2][S] reshape)."""
    L, NB = 3, 6
    lay0 = dict(L=L, H=2, D=16, e=2, bs=8, NB=NB)
    S = 8 * 2 * 16 * 2
    pool = make_pool(**lay0, kv_plane_stride=S, block_stride=2 * S)
    lay = pool.lay
    assert lay.layer_bytes == 2 * NB * S
    arena = np.zeros(4 * lay.U, np.uint8)
    pool.lend(kp.LOC_PEER, 4 * lay.U, arena)
    pool.adopt_blocks(1, [5, 0, 3])
    view = np.stack([a.reshape(NB, 2, S) for a in pool.layers])     # [L][NB][2][S]
    before = view.copy()
    pool.swap_out([1])
    img = arena.reshape(4, L, 2, S)
    for j, b in enumerate([5, 0, 3]):
        assert np.array_equal(img[j], before[:, b, :, :])
    new = pool.swap_in([1])[0]
    assert new == [0, 1, 2]
    view = np.stack([a.reshape(NB, 2, S) for a in pool.layers])
    for j, b in enumerate(new):
        assert np.array_equal(view[:, b], before[:, [5, 0, 3][j]])


def test_spec_allocation_examples():
    """SPEC S:379-381 in slots: offer 30 units; allocate 10 -> remote;
    then 25 -> DRAM fallback (20 left); no producer -> DRAM."""
    lay = kp.Layout(L=1, bs=16, H=1, D=8, e=2, NB=100)
    pool = kp.Pool(lay)
    pool.lend(kp.LOC_PEER, 30 * lay.U)
    pool.lend(kp.LOC_HOST, 1000 * lay.U)
    pool.alloc_blocks(1, 10)
    pool.alloc_blocks(2, 25)
    (r1,) = pool.swap_out([1])
    assert r1[1] == kp.LOC_PEER and len(pool.peer.free) == 20
    (r2,) = pool.swap_out([2])
    assert r2[1] == kp.LOC_HOST and len(pool.peer.free) == 20
    nopeer = kp.Pool(lay)
    nopeer.lend(kp.LOC_HOST, 1000 * lay.U)
    nopeer.alloc_blocks(3, 5)
    assert nopeer.swap_out([3])[0][1] == kp.LOC_HOST
    # nothing lent at all -> NOSPACE, no change
    bare = kp.Pool(lay)
    bare.alloc_blocks(4, 2)
    with pytest.raises(kp.AquaError) as e:
        bare.swap_out([4])
    assert e.value.code == kp.E_NOSPACE
    assert bare.query(4)[0] == kp.RESIDENT


def test_errors_are_all_or_nothing():
    pool = make_pool(NB=8)
    pool.lend(kp.LOC_PEER, 2 * pool.lay.U)
    pool.alloc_blocks(1, 2)
    pool.alloc_blocks(2, 2)
    snap = copy.deepcopy((pool.free, pool.prompts, pool.peer.free))
    cases = [
        (lambda: pool.swap_out([1, 2]), kp.E_NOSPACE),      # 2nd prompt has no room
        (lambda: pool.swap_out([1, 1]), kp.E_INVAL),
        (lambda: pool.swap_out([1, 9]), kp.E_STATE),
        (lambda: pool.swap_in([1]), kp.E_STATE),
        (lambda: pool.alloc_blocks(3, 5), kp.E_NOBLOCKS),
        (lambda: pool.alloc_blocks(3, -1), kp.E_INVAL),
        (lambda: pool.adopt_blocks(3, [0]), kp.E_INVAL),    # 0 is owned
        (lambda: pool.adopt_blocks(3, [5, 5]), kp.E_INVAL),
        (lambda: pool.adopt_blocks(3, [8]), kp.E_INVAL),
        (lambda: pool.free_prompt(42), kp.E_STATE),
    ]
    for fn, code in cases:
        with pytest.raises(kp.AquaError) as e:
            fn()
        assert e.value.code == code
        assert (pool.free, pool.prompts, pool.peer.free) == snap
    # swap_in NOBLOCKS: swap 1 out, fill the pool, try to bring it back
    pool.swap_out([1])
    pool.alloc_blocks(3, 6)
    snap = copy.deepcopy((pool.free, pool.prompts, pool.peer.free))
    with pytest.raises(kp.AquaError) as e:
        pool.swap_in([1])
    assert e.value.code == kp.E_NOBLOCKS
    assert (pool.free, pool.prompts, pool.peer.free) == snap


def test_zero_block_prompt():
    pool = make_pool(NB=4)
    pool.lend(kp.LOC_PEER, 2 * pool.lay.U)
    assert pool.alloc_blocks(5, 0) == []
    assert pool.swap_out([5]) == [(5, kp.LOC_PEER, [])]
    assert pool.swap_in([5]) == [[]]
    assert pool.query(5) == (kp.RESIDENT, kp.LOC_LOCAL, 0, [])


def test_zero_block_image_relocated_without_host_arena():
    """Reclaim moves every lender image to the host; a 0-block
    image needs no host slots, so it relocates even when no host arena was
    lent, and afterwards swap_in / free / prefix load+drop of such images
    touch no arena (found by the 3000-seed dry-run fuzz, profiles/
    r02_dry_fuzz_long.log).  Expected values hand-derived: nothing to copy,
    no slot or block changes hands."""
    pool = make_pool(L=2, NB=4)
    U = pool.lay.U
    pool.lend(kp.LOC_PEER, 2 * U, np.zeros(2 * U, np.uint8))
    assert pool.alloc_blocks(5, 0) == [] and pool.alloc_blocks(6, 0) == [] and pool.alloc_blocks(7, 2) == [0, 1]
    assert pool.prefix_store(3, 7, 0) == (kp.LOC_PEER, [])
    assert pool.swap_out([5, 6]) == [(5, kp.LOC_PEER, []), (6, kp.LOC_PEER, [])]
    before = planes(pool).copy()
    assert pool.host is None
    assert pool.reclaim() == [(5, []), (6, [])]                 # no host arena needed for 0 slots
    assert pool.peer is None and pool.query(5) == (kp.SWAPPED, kp.LOC_HOST, 0, [])
    assert (pool.prefixes[3].location, pool.prefixes[3].slots) == (kp.LOC_HOST, [])
    assert pool.swap_in([5]) == [[]]
    assert pool.query(5) == (kp.RESIDENT, kp.LOC_LOCAL, 0, [])
    pool.free_prompt(6)
    assert pool.prefix_load(3, 7) == []
    pool.prefix_drop(3)
    assert np.array_equal(planes(pool), before) and pool.free == {2, 3}
    pool.check_invariants()


# ---------------------------------------------------------------- brute force
class TinyModel:
    """Independent array-scan model of the allocator and slot placement."""

    def __init__(self, NB, nslots):
        self.blk = [None] * NB          # owner pid or None
        self.slot = [None] * nslots
        self.st = {}                    # pid -> ("R", [blocks]) | ("S", [slots])

    def _first_free(self, arr, n):
        out = [i for i, o in enumerate(arr) if o is None][:n]
        return out if len(out) == n else None

    def op(self, name, arg):
        if name == "alloc":
            pid, n = arg
            if pid in self.st and self.st[pid][0] != "R":
                return kp.E_STATE
            ids = self._first_free(self.blk, n)
            if ids is None:
                return kp.E_NOBLOCKS
            for i in ids:
                self.blk[i] = pid
            self.st.setdefault(pid, ("R", []))[1].extend(ids)
            return ids
        if name == "out":
            pid = arg
            if self.st.get(pid, ("X",))[0] != "R":
                return kp.E_STATE
            bl = self.st[pid][1]
            sl = self._first_free(self.slot, len(bl))
            if sl is None:
                return kp.E_NOSPACE
            for i in bl:
                self.blk[i] = None
            for s in sl:
                self.slot[s] = pid
            self.st[pid] = ("S", sl)
            return sl
        if name == "in":
            pid = arg
            if self.st.get(pid, ("X",))[0] != "S":
                return kp.E_STATE
            sl = self.st[pid][1]
            ids = self._first_free(self.blk, len(sl))
            if ids is None:
                return kp.E_NOBLOCKS
            for i in ids:
                self.blk[i] = pid
            for s in sl:
                self.slot[s] = None
            self.st[pid] = ("R", ids)
            return ids
        if name == "free":
            pid = arg
            if pid not in self.st:
                return kp.E_STATE
            kind, xs = self.st.pop(pid)
            for x in xs:
                (self.blk if kind == "R" else self.slot)[x] = None
            return None


def _ops(npids):
    for pid in range(npids):
        yield ("alloc", (pid, 1))
        yield ("alloc", (pid, 2))
        yield ("out", pid)
        yield ("in", pid)
        yield ("free", pid)


def _snap(pool):
    return (frozenset(pool.free), frozenset(pool.peer.free),
            {k: (v.state, v.location, tuple(v.blocks), tuple(v.slots)) for k, v in pool.prompts.items()})


@pytest.mark.parametrize("NB,nslots,length", [(3, 2, 4), (5, 3, 4), (4, 4, 3)])
def test_bruteforce_op_sequences(NB, nslots, length):
    ops = list(_ops(3))
    n = 0
    for seq in itertools.product(ops, repeat=length):
        lay = kp.Layout(L=1, bs=16, H=1, D=8, e=2, NB=NB)
        pool = kp.Pool(lay)
        pool.lend(kp.LOC_PEER, nslots * lay.U)
        ref = TinyModel(NB, nslots)
        for name, arg in seq:
            want = ref.op(name, arg)
            snap = _snap(pool)
            try:
                if name == "alloc":
                    got = pool.alloc_blocks(*arg)
                elif name == "out":
                    got = pool.swap_out([arg])[0][2]
                elif name == "in":
                    got = pool.swap_in([arg])[0]
                else:
                    got = pool.free_prompt(arg)
            except kp.AquaError as e:
                got = e.code
                assert _snap(pool) == snap
            assert got == want, (seq, name, arg)
            pool.check_invariants()
        n += 1
    assert n == len(ops) ** length


# ------------------------------------------------------------------ NEXT-1
def test_migrate_and_reclaim_bytes():
    """Images keep their bytes through lender -> host -> lender moves, and a
    resume from the new place restores the original blocks (I1 across
    migration); SPEC S:384-392 reclaim examples."""
    pool = make_pool(L=2, NB=16)
    U = pool.lay.U
    peer = np.zeros(8 * U, np.uint8)
    host = np.zeros(8 * U, np.uint8)
    pool.lend(kp.LOC_PEER, 8 * U, peer)
    pool.lend(kp.LOC_HOST, 8 * U, host)
    pool.adopt_blocks(1, [9, 2, 5])
    pool.adopt_blocks(2, [0, 1])
    before = planes(pool).copy()
    pool.swap_out([1, 2])
    img1 = peer.reshape(8, U)[[0, 1, 2]].copy()
    # reclaim: both images move to the host, ascending pid, lowest host slots
    moved = pool.reclaim()
    assert moved == [(1, [0, 1, 2]), (2, [3, 4])]
    assert pool.peer is None and pool.query(1)[1] == kp.LOC_HOST
    assert np.array_equal(host.reshape(8, U)[[0, 1, 2]], img1)
    assert pool.reclaim() == []                       # double reclaim: no-op
    # re-offer and move pid 2 back
    peer2 = np.zeros(4 * U, np.uint8)
    pool.lend(kp.LOC_PEER, 4 * U, peer2)
    assert pool.migrate([2], kp.LOC_PEER) == [(2, [0, 1])]
    assert len(pool.host.free) == 8 - 3
    new = pool.swap_in([2, 1])
    after = planes(pool)
    for pid, old in ((2, [0, 1]), (1, [9, 2, 5])):
        ids = new[0] if pid == 2 else new[1]
        for j, b in enumerate(ids):
            assert np.array_equal(after[:, :, b, :], before[:, :, old[j], :])
    pool.check_invariants()


def test_migrate_errors_all_or_nothing():
    pool = make_pool(L=1, NB=8)
    U = pool.lay.U
    pool.lend(kp.LOC_PEER, 4 * U)
    pool.lend(kp.LOC_HOST, 2 * U)
    pool.alloc_blocks(1, 2)
    pool.alloc_blocks(2, 2)
    pool.alloc_blocks(3, 1)
    pool.swap_out([1, 2])
    snap = (frozenset(pool.peer.free), frozenset(pool.host.free), pool.query(1), pool.query(2))
    for fn, code in [(lambda: pool.migrate([1, 2], kp.LOC_HOST), kp.E_NOSPACE),   # host has 2 slots
                     (lambda: pool.migrate([1], kp.LOC_PEER), kp.E_STATE),        # already there
                     (lambda: pool.migrate([3], kp.LOC_HOST), kp.E_STATE),        # resident
                     (lambda: pool.migrate([1, 1], kp.LOC_HOST), kp.E_INVAL),
                     (lambda: pool.reclaim(), kp.E_NOSPACE)]:
        with pytest.raises(kp.AquaError) as e:
            fn()
        assert e.value.code == code
        assert (frozenset(pool.peer.free), frozenset(pool.host.free), pool.query(1), pool.query(2)) == snap
    assert pool.peer is not None                      # failed reclaim keeps the lender


class TwoArenaModel:
    """Independent model with two arenas for the NEXT-1 brute force."""

    def __init__(self, NB, np_, nh):
        self.blk = [None] * NB
        self.ar = {1: [None] * np_, 2: [None] * nh}
        self.peer_on = True
        self.st = {}          # pid -> ("R", ids) | ("S", loc, slots)

    @staticmethod
    def _free(arr, n):
        out = [i for i, o in enumerate(arr) if o is None][:n]
        return out if len(out) == n else None

    def op(self, name, arg):
        if name == "alloc":
            pid, n = arg
            if pid in self.st and self.st[pid][0] != "R":
                return kp.E_STATE
            ids = self._free(self.blk, n)
            if ids is None:
                return kp.E_NOBLOCKS
            for i in ids:
                self.blk[i] = pid
            if pid not in self.st:
                self.st[pid] = ("R", [])
            self.st[pid][1].extend(ids)
            return ids
        if name == "out":
            pid = arg
            if self.st.get(pid, ("X",))[0] != "R":
                return kp.E_STATE
            ids = self.st[pid][1]
            for loc in ((1, 2) if self.peer_on else (2,)):
                sl = self._free(self.ar[loc], len(ids))
                if sl is not None:
                    break
            else:
                return kp.E_NOSPACE
            for i in ids:
                self.blk[i] = None
            for x in sl:
                self.ar[loc][x] = pid
            self.st[pid] = ("S", loc, sl)
            return (loc, sl)
        if name == "in":
            pid = arg
            if self.st.get(pid, ("X",))[0] != "S":
                return kp.E_STATE
            _, loc, sl = self.st[pid]
            ids = self._free(self.blk, len(sl))
            if ids is None:
                return kp.E_NOBLOCKS
            for i in ids:
                self.blk[i] = pid
            for x in sl:
                self.ar[loc][x] = None
            self.st[pid] = ("R", ids)
            return ids
        if name == "mig":
            pid, dst = arg
            s = self.st.get(pid, ("X",))
            if s[0] != "S" or s[1] == dst:
                return kp.E_STATE
            if dst == 1 and not self.peer_on:
                return kp.E_NOSPACE
            new = self._free(self.ar[dst], len(s[2]))
            if new is None:
                return kp.E_NOSPACE
            for x in s[2]:
                self.ar[s[1]][x] = None
            for x in new:
                self.ar[dst][x] = pid
            self.st[pid] = ("S", dst, new)
            return new
        if name == "reclaim":
            if not self.peer_on:
                return []
            pids = sorted(p for p, s in self.st.items() if s[0] == "S" and s[1] == 1)
            need = sum(len(self.st[p][2]) for p in pids)
            if need > sum(o is None for o in self.ar[2]):
                return kp.E_NOSPACE
            res = [(p, self.op("mig", (p, 2))) for p in pids]
            self.peer_on = False
            self.ar[1] = []
            return res
        if name == "relend":
            if self.peer_on:
                return kp.E_INVAL
            self.peer_on = True
            self.ar[1] = [None] * arg
            return arg


def _snap2(pool):
    return (frozenset(pool.free), None if pool.peer is None else frozenset(pool.peer.free),
            frozenset(pool.host.free),
            {k: (v.state, v.location, tuple(v.blocks), tuple(v.slots)) for k, v in pool.prompts.items()})


def test_bruteforce_with_migration():
    ops = []
    for pid in range(2):
        ops += [("alloc", (pid, 1)), ("alloc", (pid, 2)), ("out", pid), ("in", pid),
                ("mig", (pid, 1)), ("mig", (pid, 2))]
    ops += [("reclaim", None), ("relend", 3)]
    n = 0
    for seq in itertools.product(ops, repeat=4):
        lay = kp.Layout(L=1, bs=16, H=1, D=8, e=2, NB=4)
        pool = kp.Pool(lay)
        pool.lend(kp.LOC_PEER, 2 * lay.U)
        pool.lend(kp.LOC_HOST, 3 * lay.U)
        ref = TwoArenaModel(4, 2, 3)
        for name, arg in seq:
            want = ref.op(name, arg)
            snap = _snap2(pool)
            try:
                if name == "alloc":
                    got = pool.alloc_blocks(*arg)
                elif name == "out":
                    (_, loc, sl), = pool.swap_out([arg])
                    got = (loc, sl)
                elif name == "in":
                    got = pool.swap_in([arg])[0]
                elif name == "mig":
                    got = pool.migrate([arg[0]], arg[1])[0][1]
                elif name == "reclaim":
                    got = pool.reclaim()
                else:
                    got = pool.lend(kp.LOC_PEER, arg * lay.U)
            except kp.AquaError as e:
                got = e.code
                assert _snap2(pool) == snap
            assert got == want, (seq, name, arg, got, want)
            pool.check_invariants()
        n += 1
    assert n == len(ops) ** 4


# ------------------------------------------------------------------ NEXT-2
def test_prefix_cache_bytes():
    """A cached prefix is a copy: every hit gets the prefix blocks' bytes
    (checked through the layout's meaning), the source prompt and the image
    are untouched, and a reclaim moves the image with the prompts."""
    pool = make_pool(L=2, NB=32)
    U = pool.lay.U
    peer = np.zeros(8 * U, np.uint8)
    host = np.zeros(8 * U, np.uint8)
    pool.lend(kp.LOC_PEER, 8 * U, peer)
    pool.lend(kp.LOC_HOST, 8 * U, host)
    pool.adopt_blocks(5, [7, 3, 11, 0, 9])
    before = planes(pool).copy()
    assert pool.prefix_store(42, 5, 3) == (kp.LOC_PEER, [0, 1, 2])
    assert np.array_equal(planes(pool), before)                      # copy, not move
    img = peer.reshape(8, pool.lay.L, 2, pool.lay.S)
    for j, b in enumerate([7, 3, 11]):
        assert np.array_equal(img[j], before[:, :, b, :])
    hits = []
    for dst in (100, 101, 102):
        ids = pool.prefix_load(42, dst)
        hits.append(ids)
        pool.alloc_blocks(dst, 1)                                    # the suffix
    now = planes(pool)
    for ids in hits:
        for j, b in enumerate(ids):
            assert np.array_equal(now[:, :, b, :], before[:, :, [7, 3, 11][j], :])
    assert hits[0] == [1, 2, 4]                                      # lowest free after 0,3,7,9,11 taken
    pool.check_invariants()
    with pytest.raises(kp.AquaError) as e:
        pool.prefix_store(42, 5, 1)
    assert e.value.code == kp.E_INVAL
    with pytest.raises(kp.AquaError) as e:
        pool.prefix_store(43, 5, 6)
    assert e.value.code == kp.E_INVAL
    pool.swap_out([5])
    assert pool.reclaim() == [(5, [0, 1, 2, 3, 4])]
    assert pool.prefixes[42].location == kp.LOC_HOST and pool.prefixes[42].slots == [5, 6, 7]
    for j, b in enumerate([7, 3, 11]):
        assert np.array_equal(host.reshape(8, pool.lay.L, 2, pool.lay.S)[5 + j], before[:, :, b, :])
    pool.prefix_drop(42)
    pool.check_invariants()
    assert len(pool.host.free) == 3
    with pytest.raises(kp.AquaError) as e:
        pool.prefix_load(42, 200)
    assert e.value.code == kp.E_STATE


# ------------------------------------------- pins added by the mutation check
def test_lend_capacity_is_floor_of_bytes_over_U():
    """SURVEY 8(b) / include/aqua.h aqua_lend: capacity in slots =
    floor(bytes / U); a partial slot is not usable."""
    lay = kp.Layout(L=2, bs=16, H=2, D=64, e=2, NB=8)          # U = 16384
    pool = kp.Pool(lay)
    assert pool.lend(kp.LOC_PEER, 3 * lay.U + lay.U // 2) == 3
    assert pool.lend(kp.LOC_HOST, lay.U - 16) == 0
    pool.alloc_blocks(1, 1)
    with pytest.raises(kp.AquaError) as ei:                      # 0 host slots: no room
        pool.alloc_blocks(2, 4)
        pool.swap_out([2, 1])
    assert ei.value.code == kp.E_NOSPACE


def test_prefix_store_uses_a_lender_with_exactly_n_free_slots():
    """R5 for prefixes ("both CFS and prefill caching share the same
    swap space"): the lender is used when it has n free slots (>= n, not > n)."""
    lay = kp.Layout(L=1, bs=16, H=1, D=8, e=2, NB=8)
    pool = kp.Pool(lay)
    pool.lend(kp.LOC_PEER, 2 * lay.U)
    pool.lend(kp.LOC_HOST, 8 * lay.U)
    pool.alloc_blocks(7, 3)
    assert pool.prefix_store(1, 7, 2) == (kp.LOC_PEER, [0, 1])
    assert pool.prefix_store(2, 7, 1) == (kp.LOC_HOST, [0])


def test_query_reports_slots_of_a_swapped_prompt():
    """P:855-857 "the serving engine can query AquaLib for the tensor
    location": a swapped prompt reports (SWAPPED, location, n, its slots)."""
    lay = kp.Layout(L=1, bs=16, H=1, D=8, e=2, NB=8)
    pool = kp.Pool(lay)
    pool.lend(kp.LOC_PEER, 8 * lay.U)
    pool.alloc_blocks(9, 2)                                      # slots 0, 1 of a different prompt
    pool.swap_out([9])
    pool.alloc_blocks(4, 3)
    assert pool.query(4) == (kp.RESIDENT, kp.LOC_LOCAL, 3, [0, 1, 2])
    pool.swap_out([4])
    assert pool.query(4) == (kp.SWAPPED, kp.LOC_PEER, 3, [2, 3, 4])


def test_layout_chunk_must_be_16_byte_multiple():
    """SURVEY 8(a) A3 / include/aqua.h aqua_create: S = bs*H*D*e must be a
    multiple of 16 bytes (16-byte vectors and bulk copies); else INVAL."""
    with pytest.raises(kp.AquaError) as ei:
        kp.Pool(kp.Layout(L=1, bs=1, H=1, D=3, e=2, NB=4))          # S = 6 B
    assert ei.value.code == kp.E_INVAL
    kp.Pool(kp.Layout(L=1, bs=1, H=1, D=8, e=2, NB=4))              # S = 16 B is fine


def test_prefix_load_with_exactly_n_free_blocks():
    """NEXT-2 prefix load needs n free blocks: exactly n is enough (lowest
    first, R4), n - 1 is NOBLOCKS with nothing changed."""
    lay = kp.Layout(L=1, bs=16, H=1, D=8, e=2, NB=8)
    pool = kp.Pool(lay)
    pool.lend(kp.LOC_PEER, 8 * lay.U)
    pool.alloc_blocks(1, 3)                                      # blocks 0..2
    pool.prefix_store(7, 1, 3)
    pool.alloc_blocks(2, 2)                                      # 3..4: exactly 3 free (5, 6, 7)
    assert pool.prefix_load(7, 3) == [5, 6, 7]
    pool.free_prompt(3)
    pool.alloc_blocks(4, 1)                                      # 5: only 2 free
    with pytest.raises(kp.AquaError) as ei:
        pool.prefix_load(7, 5)
    assert ei.value.code == kp.E_NOBLOCKS and len(pool.free) == 2 and 5 not in pool.prompts
