"""Whole-buffer parity at BASELINE sizes (-m gpu), SURVEY 8(d) parity protocol.

* C2 (configs[1]: one 32K-token Llama-3-8B prompt, 2,048 blocks of 2 MiB) and
  C4 (configs[3] per TP rank: 32 prompts x 2,048 tokens of the 70B/TP4 shard,
  S = 8 KiB): pool and arena start as seeded random 16-bit words (not the
  pattern), the oracle runs in bytes mode on the same bytes, and the sha256
  of every pool layer and of the whole lender arena must match the oracle's
  after swap_out and again after a swap_in into a fragmented pool.  The
  arenas are 4-5 GiB, so this covers byte offsets above 2^31 (invariant I2:
  nothing outside the chosen slots / new blocks changes).
* C3 scaled down (configs[2]: the full bursty trace, seed 1, NB = 4,152,
  18,332 library calls, but a tiny KV shape): the trace driver, the native
  scheduler, the kernels and the synthetic decode on the GPU against the
  oracle's call log replayed in bytes mode; whole pool + lender + host
  arenas compared at checkpoints and at the end.

The lender is the borrower's own HBM, or GPU 1 (peer over NVLink) when the
box has two GPUs."""
import hashlib

import numpy as np
import pytest
import torch

from oracle import kvpool as kp
from oracle import sim as osim
from paper_2407_21255_b200 import aqua
from workloads import block_permutation, burst_trace, kv_random_bytes

pytestmark = pytest.mark.gpu


def _need_host_gib(g):
    try:
        import psutil
        if psutil.virtual_memory().available < (g << 30):
            pytest.skip(f"needs {g} GiB of free host memory for the bytes-mode oracle")
    except ImportError:
        pass


def _lender_dev(where):
    if where == "peer":
        if torch.cuda.device_count() < 2:
            pytest.skip("needs 2 GPUs (peer lender over NVLink)")
        return 1
    return 0


def _sha(buf) -> str:
    h = hashlib.sha256()
    h.update(memoryview(buf))
    return h.hexdigest()


def _gpu_sha(t: torch.Tensor) -> str:
    return _sha(t.cpu().numpy())


class _Big:
    """Borrower pool + lender arena on the GPU(s) and the oracle Pool, both
    from the same seeded random bytes (the numpy arrays become the oracle's
    buffers; the GPU gets a copy)."""

    def __init__(self, L, H, NB, nslots, where):
        self.lay = kp.Layout(L=L, bs=16, H=H, D=128, e=2, NB=NB)
        lb, U = self.lay.layer_bytes, self.lay.U
        dev = torch.device("cuda", 0)
        ldev = torch.device("cuda", _lender_dev(where))
        init = [kv_random_bytes(lb, seed=1000 + l) for l in range(L)]
        self.layers = [torch.from_numpy(a).to(dev) for a in init]
        self.opool = kp.Pool(self.lay, init)
        a = kv_random_bytes(nslots * U, seed=77)
        self.arena = torch.from_numpy(a).to(ldev)
        self.opool.lend(kp.LOC_PEER, nslots * U, a)
        self.ctx = aqua.Ctx(0, L, 16, H, 128, 2, NB, [t.data_ptr() for t in self.layers])
        assert self.ctx.lend(ldev.index, self.arena.data_ptr(), nslots * U) == nslots
        info = self.ctx.arena_info(aqua.LOC_PEER)
        assert info["peer"] == (where == "peer") and info["device"] == ldev.index

    def compare(self, what):
        torch.cuda.synchronize()
        bad = [l for l, t in enumerate(self.layers) if _gpu_sha(t) != _sha(self.opool.layers[l])]
        assert not bad, f"{what}: pool layers {bad[:8]} differ from the oracle"
        assert _gpu_sha(self.arena) == _sha(self.opool.peer.data), f"{what}: lender arena differs"

    def close(self):
        self.ctx.close()


@pytest.mark.parametrize("where", ["self", "peer"])
def test_c2_whole_buffer_sha256(where):
    _need_host_gib(20)
    B = _Big(L=32, H=8, NB=4096, nslots=2048, where=where)
    c, o = B.ctx, B.opool
    perm = block_permutation(4096, 4096, seed=2).tolist()
    bt = perm[:2048]
    c.adopt_blocks(7, bt)
    o.adopt_blocks(7, bt)
    c.adopt_blocks(8, perm[2048:])            # filler: the free set after swap_out is scattered
    o.adopt_blocks(8, perm[2048:])
    c.swap_out([7])
    o.swap_out([7])
    assert c.query(7, with_ids=True)[1:] == (kp.LOC_PEER, 2048, list(range(2048)))
    B.compare("after swap_out")
    # fragment the pool, then resume into whatever is left
    ids = c.alloc_blocks(9, 700)
    assert ids == o.alloc_blocks(9, 700)
    c.free(8)
    o.free_prompt(8)
    new, _ = c.swap_in([7])
    assert new == o.swap_in([7])
    assert new[0] != list(range(new[0][0], new[0][0] + 2048))
    B.compare("after swap_in into a fragmented pool")
    B.close()


@pytest.mark.parametrize("where", ["self", "peer"])
def test_c4_whole_buffer_sha256(where):
    _need_host_gib(24)
    NB, nblk = 8192, 4096
    B = _Big(L=80, H=2, NB=NB, nslots=nblk, where=where)
    c, o = B.ctx, B.opool
    perm = block_permutation(NB, NB, seed=2).tolist()
    c.adopt_blocks(1, perm[nblk:])
    o.adopt_blocks(1, perm[nblk:])
    pids = list(range(100, 132))
    for i, pid in enumerate(pids):
        c.adopt_blocks(pid, perm[i * 128:(i + 1) * 128])
        o.adopt_blocks(pid, perm[i * 128:(i + 1) * 128])
    c.swap_out(pids)                          # one call, 4,096 descriptors
    o.swap_out(pids)
    B.compare("after swap_out")
    c.free(1)
    o.free_prompt(1)
    assert c.alloc_blocks(2, 3000) == o.alloc_blocks(2, 3000)
    new, _ = c.swap_in(pids[::-1])
    assert new == o.swap_in(pids[::-1])
    B.compare("after swap_in into a fragmented pool")
    B.close()


def test_c3_scaled_whole_buffer_vs_oracle_bytes():
    """configs[2]'s full trace (seed 1, NB = 4,152, lender and host arenas of
    32,768 slots) with a tiny KV shape (L=2, H=2, D=64: U = 16 KiB): the GPU
    run (Python trace driver + native scheduler + libaqua kernels + the
    synthetic decode kernel) and the oracle (sim.run's call log replayed in
    bytes mode) hold identical pool, lender and host bytes at every
    checkpoint."""
    from paper_2407_21255_b200.cfs import Scheduler
    from paper_2407_21255_b200.driver import run_trace
    _need_host_gib(4)
    L, bs, H, D, NB, NS, SEED = 2, 16, 2, 64, 4152, 32768, 77
    tr = burst_trace(seed=1)
    lay = kp.Layout(L=L, bs=bs, H=H, D=D, e=2, NB=NB)
    init = [kv_random_bytes(lay.layer_bytes, seed=l) for l in range(L)]
    peer0 = kv_random_bytes(NS * lay.U, seed=100)
    host0 = kv_random_bytes(NS * lay.U, seed=200)
    dev = torch.device("cuda", 0)
    layers = [torch.from_numpy(a.copy()).to(dev) for a in init]
    arena = torch.from_numpy(peer0.copy()).to(dev)
    host = torch.from_numpy(host0.copy()).pin_memory()
    c = aqua.Ctx(0, L, bs, H, D, 2, NB, [t.data_ptr() for t in layers])
    c.lend(0, arena.data_ptr(), NS * lay.U)
    c.lend(aqua.HOST, host.data_ptr(), NS * lay.U)
    every = 500
    got = {}

    def snap(i, work):
        if i % every == 0:
            torch.cuda.synchronize()
            got[i] = ([_gpu_sha(t) for t in layers], _gpu_sha(arena), _sha(host.numpy()))

    log, st = run_trace(tr, c, Scheduler(NB=NB, bs=bs, b=512, k=8), fill_seed=SEED, on_iteration=snap)
    torch.cuda.synchronize()
    final = ([_gpu_sha(t) for t in layers], _gpu_sha(arena), _sha(host.numpy()))
    c.close()

    o = osim.run(tr, osim.SimConfig(NB=NB, lender_slots=NS, host_slots=NS))
    assert log == o.log and st["blocks_out"] == o.blocks_out > 0
    pool = kp.Pool(lay, init)
    pool.lend(kp.LOC_PEER, NS * lay.U, peer0)
    pool.lend(kp.LOC_HOST, NS * lay.U, host0)
    want = {}

    def osnap(i):
        if i % every == 0:
            want[i] = ([_sha(a) for a in pool.layers], _sha(pool.peer.data), _sha(pool.host.data))

    osim.replay_bytes(o.log, pool, SEED, on_iter=osnap)
    assert sorted(got) == sorted(want) and len(got) >= 10
    for i in sorted(got):
        assert got[i] == want[i], f"bytes differ at iteration {i}"
    assert final == ([_sha(a) for a in pool.layers], _sha(pool.peer.data), _sha(pool.host.data))
