"""Shared helpers for the -m gpu parity tests: device buffers filled from the
seeded generators, and an oracle Pool holding the same initial bytes."""
import weakref

import numpy as np
import torch

from oracle import kvpool as kp
from paper_2407_21255_b200 import aqua
from workloads import kv_random_bytes


class Rig:
    """A borrower pool (L device tensors), a GPU lender arena (caller-owned
    device tensor) and a pinned host arena, mirrored by an oracle Pool with
    identical initial bytes.  Every Rig's ctx is destroyed after its test
    (tests/conftest.py), so a leak check sees the library free everything."""
    live = weakref.WeakSet()

    def __init__(self, L=2, bs=16, H=2, D=64, e=2, NB=40, lender_slots=12, host_slots=0, seed=0,
                 kv_plane_stride=0, block_stride=0, device=0, lender_device=None, peer_test=0):
        self.lay = kp.Layout(L=L, bs=bs, H=H, D=D, e=e, NB=NB,
                             kv_plane_stride=kv_plane_stride or None, block_stride=block_stride or None)
        lb = self.lay.layer_bytes
        init = [kv_random_bytes(lb + (lb & 1), seed=seed + l)[:lb].copy() for l in range(L)]
        self.dev = torch.device("cuda", device)
        self.layers = [torch.from_numpy(a.copy()).to(self.dev) for a in init]
        self.opool = kp.Pool(self.lay, [a.copy() for a in init])
        U = self.lay.U
        self.ctx = aqua.Ctx(device, L, bs, H, D, e, NB, [t.data_ptr() for t in self.layers],
                            kv_plane_stride, block_stride)
        Rig.live.add(self)
        self.peer = self.host = None
        if peer_test:
            self.ctx.set_option(aqua.OPT_PEER_TEST, peer_test)
        if lender_slots:
            g = kv_random_bytes(lender_slots * U, seed=100 + seed)
            ldev = torch.device("cuda", device if lender_device is None else lender_device)
            self.peer = torch.from_numpy(g.copy()).to(ldev)
            self.opool.lend(kp.LOC_PEER, lender_slots * U, g.copy())
            self.ctx.lend(ldev.index, self.peer.data_ptr(), lender_slots * U)
        if host_slots:
            h = kv_random_bytes(host_slots * U, seed=200 + seed)
            self.host = torch.from_numpy(h.copy()).pin_memory()
            self.opool.lend(kp.LOC_HOST, host_slots * U, h.copy())
            self.ctx.lend(aqua.HOST, self.host.data_ptr(), host_slots * U)

    def assert_bytes_equal(self, what=""):
        torch.cuda.synchronize()
        for l, t in enumerate(self.layers):
            got = t.cpu().numpy()
            want = self.opool.layers[l]
            if not np.array_equal(got, want):
                bad = np.flatnonzero(got != want)
                raise AssertionError(f"{what}: layer {l} differs at {bad.size} bytes, first {bad[:8]}")
        if self.peer is not None:
            assert np.array_equal(self.peer.cpu().numpy(), self.opool.peer.data), f"{what}: lender arena differs"
        if self.host is not None:
            assert np.array_equal(self.host.numpy(), self.opool.host.data), f"{what}: host arena differs"


def close_all():
    """Destroy every live Rig's context (the conftest fixture runs this after each test)."""
    for r in list(Rig.live):
        r.ctx.close()
