"""The peer-lender (NVLink) path (-m gpu): the lender's HBM belongs to another
GPU and the borrower's kernels store into it (swap_out) and load from it
(swap_in pull) directly -- the paper's context switch to a producer GPU's
memory (Sec. 7; testbed with NVLink).

* On any box: the peer policy through the AQUA_OPT_PEER_TEST hook, which makes
  libaqua treat a same-GPU arena as a peer: the lend-time probe (plain, bulk
  store and bulk load round trips that restore the arena's bytes), the peer
  CTA cap, and the LDST fallback when the bulk-copy probe fails -- bytes
  identical to the oracle in every case.
* With >= 2 GPUs (skipped otherwise): C1 and random op sequences with the
  lender on GPU 1 for every product engine, whole-buffer equality with the
  oracle after every call."""
import json
import os
import random

import pytest
import torch

from oracle import kvpool as kp
from paper_2407_21255_b200 import aqua
from workloads import block_permutation

from gpu_util import Rig

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")

two_gpus = pytest.mark.skipif(torch.cuda.is_available() and torch.cuda.device_count() < 2,
                              reason="needs 2 GPUs (peer lender over NVLink)")


def _roundtrip(rig, nblk, pid=5):
    c, o = rig.ctx, rig.opool
    perm = block_permutation(rig.lay.NB, nblk, seed=3).tolist()
    c.adopt_blocks(pid, perm)
    o.adopt_blocks(pid, perm)
    c.swap_out([pid])
    o.swap_out([pid])
    out_launch = c.last_launch()
    rig.assert_bytes_equal("peer swap_out")
    assert c.alloc_blocks(6, 7) == o.alloc_blocks(6, 7)
    new, _ = c.swap_in([pid])
    assert new == o.swap_in([pid])
    in_launch = c.last_launch()
    rig.assert_bytes_equal("peer swap_in")
    for p in (pid, 6):
        c.free(p)
        o.free_prompt(p)
    return out_launch, in_launch


@pytest.mark.parametrize("mode", [1, 2])
def test_peer_policy_via_test_hook(mode):
    """mode 1: a healthy peer -> probe 7, TMA engine capped at the peer CTA
    cap (default 32); mode 2: bulk copies 'fail' the probe -> LDST engine.
    The probe leaves the arena's bytes unchanged (whole-buffer check)."""
    rig = Rig(L=4, bs=16, H=8, D=128, NB=600, lender_slots=520, host_slots=0, peer_test=mode)
    info = rig.ctx.arena_info(aqua.LOC_PEER)
    assert info["peer"] and info["probe"] == (7 if mode == 1 else 1) and info["nslots"] == 520
    rig.assert_bytes_equal("after the lend-time probe")
    assert rig.ctx.get_option(aqua.OPT_PEER_CTAS) == 32
    lo, li = _roundtrip(rig, 512)
    for launch in (lo, li):
        assert launch["engine"] == ("tma" if mode == 1 else "ldst")
        assert launch["ctas"] <= 32
    # the cap can be lifted (0 = all SMs) or tightened
    rig.ctx.set_option(aqua.OPT_PEER_CTAS, 0)
    lo, _ = _roundtrip(rig, 512, pid=8)
    assert lo["ctas"] > 32
    rig.ctx.set_option(aqua.OPT_PEER_CTAS, 8)
    lo, _ = _roundtrip(rig, 512, pid=9)
    assert lo["ctas"] <= 8
    rig.ctx.close()


def test_local_lender_is_not_a_peer():
    rig = Rig(L=2, bs=16, H=2, D=64, NB=40, lender_slots=12)
    info = rig.ctx.arena_info(aqua.LOC_PEER)
    assert info == {"device": 0, "peer": False, "probe": -1, "nslots": 12}
    rig.ctx.close()


@two_gpus
@pytest.mark.parametrize("engine", ["auto", "tma", "tma_hybrid", "ldst"])
@pytest.mark.parametrize("variant", ["lender12", "lender8"])
def test_c1_bytes_peer_lender(engine, variant):
    from test_gpu_parity import _engine, _ops
    g = json.load(open(os.path.join(GOLD, "c1_script.json")))
    v = g[variant]
    rig = Rig(**g["layout"], lender_slots=v["lender_slots"], host_slots=v.get("host_slots", 0), lender_device=1)
    info = rig.ctx.arena_info(aqua.LOC_PEER)
    assert info["peer"] and info["device"] == 1 and info["probe"] == 7
    if engine != "auto":
        _engine(rig.ctx, engine)
    ops = [("alloc", (p, 4)) for p in range(8)]
    ops += [("out", g["swap_out"]), ("alloc", (100, 6)), ("in", g["swap_in"]), ("free", 100)]
    _ops(rig, ops, stream=torch.cuda.Stream().cuda_stream)
    for pid, ids in g["expected_swap_in_ids"].items():
        assert rig.ctx.query(int(pid), with_ids=True)[3] == ids


@two_gpus
@pytest.mark.parametrize("shape", ["c4_shape", "llama_bs32", "s2k", "ragged_10KiB"])
@pytest.mark.parametrize("engine", ["auto", "tma_hybrid", "ldst"])
@pytest.mark.parametrize("seed", [0, 1])
def test_random_sequences_peer_lender(shape, engine, seed):
    from test_gpu_parity import SHAPES, _engine, _ops
    L, bs, H, D, *e = SHAPES[shape]
    rnd = random.Random(seed * 17 + len(shape))
    rig = Rig(L=L, bs=bs, H=H, D=D, e=(e or [2])[0], NB=24, lender_slots=10, host_slots=8, seed=seed,
              lender_device=1)
    if engine != "auto":
        _engine(rig.ctx, engine)
    pids = list(range(5))
    for _ in range(25):
        k = rnd.random()
        p = rnd.choice(pids)
        if k < 0.35:
            op = ("alloc", (p, rnd.randint(0, 4)))
        elif k < 0.6:
            op = ("out", rnd.sample(pids, rnd.randint(1, 3)))
        elif k < 0.85:
            op = ("in", rnd.sample(pids, rnd.randint(1, 3)))
        else:
            op = ("free", p)
        try:
            _ops(rig, [op])
        except (kp.AquaError, aqua.AquaError) as e:
            # errors must agree and change nothing on either side
            code_o = code_c = None
            name, arg = op
            try:
                {"alloc": lambda: rig.opool.alloc_blocks(*arg), "out": lambda: rig.opool.swap_out(arg),
                 "in": lambda: rig.opool.swap_in(arg), "free": lambda: rig.opool.free_prompt(arg)}[name]()
            except kp.AquaError as eo:
                code_o = eo.code
            try:
                {"alloc": lambda: rig.ctx.alloc_blocks(*arg), "out": lambda: rig.ctx.swap_out(arg),
                 "in": lambda: rig.ctx.swap_in(arg, cap=4096), "free": lambda: rig.ctx.free(arg)}[name]()
            except aqua.AquaError as ec:
                code_c = ec.code
            assert code_o is not None and code_o == code_c == e.code, (op, code_o, code_c)
            rig.assert_bytes_equal(f"after failed {op}")


@two_gpus
def test_peer_exchange_and_migration_bytes():
    """Both link directions in one call (aqua_swap_exchange) and lender <->
    host migration with the lender on GPU 1."""
    rig = Rig(L=3, bs=16, H=2, D=64, NB=64, lender_slots=24, host_slots=24, lender_device=1)
    c, o = rig.ctx, rig.opool
    for p in range(4):
        assert c.alloc_blocks(p, 6) == o.alloc_blocks(p, 6)
    c.swap_out([0, 1])
    o.swap_out([0, 1])
    rig.assert_bytes_equal("swap_out")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    new, _, _ = c.swap_exchange([2, 3], [1, 0], s1.cuda_stream, s2.cuda_stream, 4)
    o.swap_out([2, 3])
    assert new == o.swap_in([1, 0])
    rig.assert_bytes_equal("exchange")
    c.migrate([2], aqua.LOC_HOST)
    o.migrate([2], kp.LOC_HOST)
    rig.assert_bytes_equal("migrate to host")
    c.migrate([2], aqua.LOC_PEER)
    o.migrate([2], kp.LOC_PEER)
    rig.assert_bytes_equal("migrate back to the peer")


@pytest.mark.parametrize("shape", ["c4_shape", "s2k", "ragged_10KiB", "s512"])
@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("seed", [0, 1])
def test_random_sequences_peer_policy_one_gpu(shape, mode, seed):
    """The peer path's host logic on any box: random alloc / swap_out /
    swap_in / free / migrate sequences against a same-GPU arena treated as a
    peer (mode 1: TMA capped at 32 CTAs; mode 2: bulk probe failed -> LDST),
    whole-buffer equality with the oracle after every call, and errors that
    agree and change nothing."""
    from test_gpu_parity import SHAPES, _ops
    L, bs, H, D, *e = SHAPES[shape]
    rnd = random.Random(seed * 7 + mode + len(shape))
    rig = Rig(L=L, bs=bs, H=H, D=D, e=(e or [2])[0], NB=24, lender_slots=10, host_slots=8, seed=seed,
              peer_test=mode)
    assert rig.ctx.arena_info(aqua.LOC_PEER)["probe"] == (7 if mode == 1 else 1)
    c, o = rig.ctx, rig.opool
    pids = list(range(5))
    for _ in range(30):
        k = rnd.random()
        p = rnd.choice(pids)
        if k < 0.3:
            op = ("alloc", (p, rnd.randint(0, 4)))
        elif k < 0.55:
            op = ("out", rnd.sample(pids, rnd.randint(1, 3)))
        elif k < 0.8:
            op = ("in", rnd.sample(pids, rnd.randint(1, 3)))
        elif k < 0.9:
            op = ("mig", (rnd.sample(pids, rnd.randint(1, 2)), rnd.choice([aqua.LOC_PEER, aqua.LOC_HOST])))
        else:
            op = ("free", p)
        name, arg = op
        # does the call move an image to or from the (pretend) peer arena?
        on_peer = lambda ps: any(q in o.prompts and o.prompts[q].location == kp.LOC_PEER for q in ps)
        # a call with images in both arenas is split (AUTO): its last launch is the copy engines' local gather
        locs = lambda ps: {o.prompts[q].location for q in ps if q in o.prompts}
        try:
            touches = name == "in" and on_peer(arg)     # a migration runs on the copy engines: no launch
            n0 = c.launch_count()
            mixed = name == "in" and {kp.LOC_PEER, kp.LOC_HOST} <= locs(arg)
            if name == "mig":
                c.migrate(arg[0], arg[1])
                o.migrate(arg[0], arg[1])
                rig.assert_bytes_equal(f"after {op}")
            else:
                _ops(rig, [op])
            touches = touches or (name == "out" and on_peer(arg))
            mixed = mixed or (name == "out" and {kp.LOC_PEER, kp.LOC_HOST} <= locs(arg))
            if name == "mig":
                assert c.launch_count() == n0
            if touches and not mixed:
                launch = c.last_launch()
                assert launch["ctas"] <= 32 and launch["engine"] == ("tma" if mode == 1 else "ldst"), launch
        except (kp.AquaError, aqua.AquaError) as err:
            code_o = code_c = None
            call_o = {"alloc": lambda: o.alloc_blocks(*arg), "out": lambda: o.swap_out(arg),
                      "in": lambda: o.swap_in(arg), "free": lambda: o.free_prompt(arg),
                      "mig": lambda: o.migrate(arg[0], arg[1])}[name]
            call_c = {"alloc": lambda: c.alloc_blocks(*arg), "out": lambda: c.swap_out(arg),
                      "in": lambda: c.swap_in(arg, cap=4096), "free": lambda: c.free(arg),
                      "mig": lambda: c.migrate(arg[0], arg[1])}[name]
            try:
                call_o()
            except kp.AquaError as eo:
                code_o = eo.code
            try:
                call_c()
            except aqua.AquaError as ec:
                code_c = ec.code
            assert code_o is not None and code_o == code_c, (op, code_o, code_c, err)
            rig.assert_bytes_equal(f"after failed {op}")
