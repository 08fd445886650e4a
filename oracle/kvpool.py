"""Oracle: paged KV pool, block allocator, swap arenas, swap_out / swap_in.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): never imported by the
product path.

What the paper fixes (arXiv 2407.21255):
  * P:842-845 (Sec. 7, "Efficient context switching"): "vLLM stores the
    key-value tensors of all the prompts associated with a layer as one
    tensor", so one prompt's K/V is scattered over per-layer tensors.
  * swap-out gathers those small pieces and copies them into the
    offloaded AquaTensor; swap-in copies the offloaded data back and
    scatters it "to respective smaller tensors".  Pure byte movement: the
    result of swap-out-then-swap-in is the original bytes (the method
    reaches exactly the plain definition, so this oracle IS that definition).
  * P:668-676 (fig:aqua_design caption) + P:749-753 (Sec. 6 "Allocating"):
    swap space lives on the paired producer GPU; "if no producer GPUs exist
    ... falls back to using the DRAM"; "If GPU 0 only has enough memory to
    offload one tensor, AquaLib falls back to the host DRAM".
  * P:529-534 (Sec. 5): one producer per consumer.
  * allocation is all-or-nothing, paired producer first,
    else DRAM.

Readings where the paper is silent (numbered as in DESIGN.md "Readings"):
  R1  KV layout: vLLM v0.5.3 flash layout per layer [2][NB][bs][H][D],
      generalised by two byte strides (kv_plane_stride, block_stride).
  R3  swap image layout: slot-major, slot s = bytes [s*U, (s+1)*U) of the
      arena, chunk (l, kv) at offset (2*l + kv)*S inside the slot.
  R4  block allocator: the n lowest free ids, ascending; call order.
  R5  placement: whole prompt in one place; paired lender first, then the
      host arena, else the whole call fails (NOSPACE).
  R6  whole blocks are copied (the tail of a partly-filled last block too).
  R7  reuse timing: sequential semantics (the GPU path must be equivalent).

Sizes: S = bs*H*D*e bytes per (layer, K|V, block) chunk; U = 2*L*S bytes
per block across all layers and K/V (the unit of work).
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Sequence

import numpy as np

# Status codes -- the values of the C ABI (include/aqua.h) so that tests can
# compare error behaviour; the oracle does not read the header.
OK = 0
E_INVAL = -1
E_NOBLOCKS = -2
E_NOSPACE = -3
E_STATE = -4

RESIDENT = 1
SWAPPED = 2

LOC_LOCAL = 0   # blocks in the borrower's own pool
LOC_PEER = 1    # image on the paired lender GPU ("pink box 1")
LOC_HOST = 2    # image in pinned host DRAM ("pink box 2")


class AquaError(Exception):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"{code}: {msg}")
        self.code = code


@dataclasses.dataclass(frozen=True)
class Layout:
    """C-1 / R1. L layers, bs tokens per block, H KV heads, D head dim,
    e element bytes, NB blocks in the pool.  Strides are in bytes."""
    L: int
    bs: int
    H: int
    D: int
    e: int
    NB: int
    kv_plane_stride: Optional[int] = None   # default NB*S (flash layout)
    block_stride: Optional[int] = None      # default S

    @property
    def S(self) -> int:
        return self.bs * self.H * self.D * self.e

    @property
    def U(self) -> int:
        return 2 * self.L * self.S

    @property
    def P_kv(self) -> int:
        return self.NB * self.S if self.kv_plane_stride is None else self.kv_plane_stride

    @property
    def P_b(self) -> int:
        return self.S if self.block_stride is None else self.block_stride

    @property
    def layer_bytes(self) -> int:
        """Smallest per-layer tensor that holds every chunk."""
        return self.P_kv + (self.NB - 1) * self.P_b + self.S


@dataclasses.dataclass
class Prompt:
    state: int
    blocks: List[int]          # block table while RESIDENT
    location: int              # LOC_* of the bytes
    slots: List[int]           # swap slots while SWAPPED


class Arena:
    """C-3: a swap arena of nslots slots of U bytes (lender HBM or host)."""

    def __init__(self, nslots: int, data: Optional[np.ndarray]):
        self.nslots = nslots
        self.free = set(range(nslots))
        self.data = data  # uint8[nslots*U] or None in metadata mode


class Pool:
    """The borrower's paged KV pool plus its swap arenas (one ctx of the
    C ABI).  ``layers`` = L uint8 arrays of layout.layer_bytes (bytes mode)
    or None (metadata mode: ids / states / slots only)."""

    def __init__(self, layout: Layout, layers: Optional[Sequence[np.ndarray]] = None):
        if layout.S % 16 != 0:
            raise AquaError(E_INVAL, "S must be a multiple of 16 bytes")
        self.lay = layout
        self.layers = list(layers) if layers is not None else None
        if self.layers is not None:
            assert len(self.layers) == layout.L
            for a in self.layers:
                assert a.dtype == np.uint8 and a.size >= layout.layer_bytes
        self.free = set(range(layout.NB))          # C-2 free block set
        self.prompts: Dict[int, Prompt] = {}
        self.prefixes: Dict[int, Prompt] = {}      # NEXT-2 persistent images
        self.peer: Optional[Arena] = None
        self.host: Optional[Arena] = None

    # ---------------------------------------------------------------- C-1
    def chunk(self, l: int, kv: int, b: int) -> np.ndarray:
        """View of chunk (l, kv, b): bytes [kv*P_kv + b*P_b, +S) of layer l."""
        lay = self.lay
        off = kv * lay.P_kv + b * lay.P_b
        return self.layers[l][off:off + lay.S]

    # ---------------------------------------------------------------- C-3
    def lend(self, kind: int, nbytes: int, data: Optional[np.ndarray] = None) -> int:
        """aqua_lend: register swap space; capacity = floor(bytes / U) slots.
        At most one peer lender and one host arena."""
        nslots = nbytes // self.lay.U
        if kind == LOC_PEER:
            if self.peer is not None:
                raise AquaError(E_INVAL, "one peer lender per borrower")
            self.peer = Arena(nslots, data)
        elif kind == LOC_HOST:
            if self.host is not None:
                raise AquaError(E_INVAL, "one host arena per borrower")
            self.host = Arena(nslots, data)
        else:
            raise AquaError(E_INVAL, "kind")
        return nslots

    def arena(self, loc: int) -> Optional[Arena]:
        return self.peer if loc == LOC_PEER else self.host

    # ---------------------------------------------------------------- C-2
    def _take_lowest(self, n: int) -> List[int]:
        """R4: remove and return the n smallest free block ids, ascending."""
        ids = sorted(self.free)[:n]
        for b in ids:
            self.free.remove(b)
        return ids

    def alloc_blocks(self, pid: int, n: int) -> List[int]:
        """Append n fresh blocks to pid (creating it RESIDENT)."""
        if n < 0:
            raise AquaError(E_INVAL, "n < 0")
        p = self.prompts.get(pid)
        if p is not None and p.state != RESIDENT:
            raise AquaError(E_STATE, "pid swapped")
        if len(self.free) < n:
            raise AquaError(E_NOBLOCKS, "pool exhausted")
        ids = self._take_lowest(n)
        if p is None:
            p = self.prompts[pid] = Prompt(RESIDENT, [], LOC_LOCAL, [])
        p.blocks.extend(ids)
        return ids

    def adopt_blocks(self, pid: int, ids: Sequence[int]) -> None:
        """Append caller-chosen block ids, in the given order; every id must
        be in range, free and distinct, else INVAL with no change."""
        ids = [int(x) for x in ids]
        if len(set(ids)) != len(ids) or any(not (0 <= b < self.lay.NB) for b in ids) \
                or any(b not in self.free for b in ids):
            raise AquaError(E_INVAL, "ids not free/distinct")
        p = self.prompts.get(pid)
        if p is not None and p.state != RESIDENT:
            raise AquaError(E_STATE, "pid swapped")
        for b in ids:
            self.free.remove(b)
        if p is None:
            p = self.prompts[pid] = Prompt(RESIDENT, [], LOC_LOCAL, [])
        p.blocks.extend(ids)

    # ---------------------------------------------------------------- C-4
    def swap_out(self, pids: Sequence[int]) -> List[tuple]:
        """Preempt ("paging out prompts that are not a part of the
        next batch"; P:849-851 gather then copy to the AquaTensor).

        Validation first, all-or-nothing: every pid known, RESIDENT, listed
        once; placement of every prompt decided in call order (R5) before
        anything changes.  Then, per prompt, per block j (block-table order)
        with b = bt[j] and slot s = slots[j], per layer l and kv in {K, V}:
            arena[s*U + (2l+kv)*S : +S] = chunk(l, kv, b)
        Then the blocks go back to the free set; the prompt is SWAPPED.
        Returns [(pid, location, slots)] in call order."""
        lay = self.lay
        pids = [int(p) for p in pids]
        if len(set(pids)) != len(pids):
            raise AquaError(E_INVAL, "duplicate pid")
        for pid in pids:
            p = self.prompts.get(pid)
            if p is None or p.state != RESIDENT:
                raise AquaError(E_STATE, f"pid {pid} not resident")
        # placement (R5), tentatively
        peer_free = sorted(self.peer.free) if self.peer else None
        host_free = sorted(self.host.free) if self.host else None
        plan = []
        for pid in pids:
            n = len(self.prompts[pid].blocks)
            if peer_free is not None and len(peer_free) >= n:
                plan.append((pid, LOC_PEER, peer_free[:n]))
                peer_free = peer_free[n:]
            elif host_free is not None and len(host_free) >= n:
                plan.append((pid, LOC_HOST, host_free[:n]))
                host_free = host_free[n:]
            else:
                raise AquaError(E_NOSPACE, f"no swap space for pid {pid}")
        # commit: copy bytes, release blocks
        for pid, loc, slots in plan:
            p = self.prompts[pid]
            ar = self.arena(loc)
            for s in slots:
                ar.free.remove(s)
            if self.layers is not None and ar.data is not None:
                for j, (b, s) in enumerate(zip(p.blocks, slots)):
                    for l in range(lay.L):
                        for kv in (0, 1):
                            off = s * lay.U + (2 * l + kv) * lay.S
                            ar.data[off:off + lay.S] = self.chunk(l, kv, b)
            self.free.update(p.blocks)
            p.blocks = []
            p.state, p.location, p.slots = SWAPPED, loc, list(slots)
        return [(pid, loc, list(slots)) for pid, loc, slots in plan]

    # ---------------------------------------------------------------- C-5
    def swap_in(self, pids: Sequence[int]) -> List[List[int]]:
        """Resume ("paging in prompts that were not on the GPU";
        P:851-853 copy back and scatter).

        All-or-nothing: every pid SWAPPED and listed once, and the pool has
        sum(n_p) free blocks.  Per prompt in call order: new = the n_p lowest
        free blocks (R4); per j, l, kv:
            chunk(l, kv, new[j]) = arena[slots[j]*U + (2l+kv)*S : +S]
        Then the slots go back to their arena; the prompt is RESIDENT with
        block table ``new``.  Returns the new block tables in call order."""
        lay = self.lay
        pids = [int(p) for p in pids]
        if len(set(pids)) != len(pids):
            raise AquaError(E_INVAL, "duplicate pid")
        for pid in pids:
            p = self.prompts.get(pid)
            if p is None or p.state != SWAPPED:
                raise AquaError(E_STATE, f"pid {pid} not swapped")
        need = sum(len(self.prompts[pid].slots) for pid in pids)
        if need > len(self.free):
            raise AquaError(E_NOBLOCKS, "pool exhausted")
        out = []
        for pid in pids:
            p = self.prompts[pid]
            new = self._take_lowest(len(p.slots))
            ar = self.arena(p.location)      # None only for a 0-block image relocated by reclaim
            if p.slots and self.layers is not None and ar.data is not None:
                for j, (b, s) in enumerate(zip(new, p.slots)):
                    for l in range(lay.L):
                        for kv in (0, 1):
                            off = s * lay.U + (2 * l + kv) * lay.S
                            self.chunk(l, kv, b)[:] = ar.data[off:off + lay.S]
            if p.slots:
                ar.free.update(p.slots)
            p.state, p.location, p.slots, p.blocks = RESIDENT, LOC_LOCAL, [], new
            out.append(list(new))
        return out

    # ---------------------------------------------------------- NEXT-1
    def migrate(self, pids: Sequence[int], dst: int) -> List[tuple]:
        """Move swap images between arenas (NEXT-1).  Paper Sec. 6
        "Reclaiming AquaTensors": a producer whose load rises
        takes its memory back and the consumer's tensors must move off it;
        when the load falls the memory is offered again and AquaLib "moves
        the offloaded tensors of the consumer back to the producer's GPU"
        (fig:elastic_result).  SPEC migrate S:399-407.

        All-or-nothing: pids listed once, each SWAPPED and not already in
        `dst`, the dst arena present with room for all of them.  Per prompt
        in call order: new = the n_p lowest free dst slots (R4); per j:
            dst[new_j*U : +U] = src[old_j*U : +U]
        then the old slots are freed.  Returns [(pid, new_slots)]."""
        pids = [int(p) for p in pids]
        if dst not in (LOC_PEER, LOC_HOST) or len(set(pids)) != len(pids):
            raise AquaError(E_INVAL, "bad dst or duplicate pid")
        for pid in pids:
            p = self.prompts.get(pid)
            if p is None or p.state != SWAPPED or p.location == dst:
                raise AquaError(E_STATE, f"pid {pid} has no image outside dst")
        ar_d = self.arena(dst)
        if ar_d is None:
            raise AquaError(E_NOSPACE, "no such arena")
        need = sum(len(self.prompts[pid].slots) for pid in pids)
        if need > len(ar_d.free):
            raise AquaError(E_NOSPACE, "dst arena full")
        return [(pid, slots) for pid, slots in zip(pids, self._move([self.prompts[p] for p in pids], dst))]

    def _move(self, images: List[Prompt], dst: int) -> List[List[int]]:
        """Copy each image to the lowest free dst slots, in order; free the
        old slots.  (Capacity already checked by the caller.)"""
        lay = self.lay
        ar_d = self.arena(dst)
        out = []
        for p in images:
            ar_s = self.arena(p.location)
            new = sorted(ar_d.free)[:len(p.slots)] if p.slots else []   # a 0-block image only relocates
            for s in new:
                ar_d.free.remove(s)
            if p.slots and ar_s.data is not None and ar_d.data is not None:
                for s_old, s_new in zip(p.slots, new):
                    ar_d.data[s_new * lay.U:(s_new + 1) * lay.U] = ar_s.data[s_old * lay.U:(s_old + 1) * lay.U]
            if p.slots:
                ar_s.free.update(p.slots)
            p.location, p.slots = dst, list(new)
            out.append(list(new))
        return out

    def reclaim(self) -> List[tuple]:
        """The GPU lender takes its memory back: every image on
        it moves to the host arena -- prompts in ascending pid, then cached
        prefixes in ascending id -- and the lender is detached (a later
        lend() is a re-offer).  All-or-nothing (NOSPACE if the host
        cannot hold them); idempotent without a lender ("double
        reclaim -> no-op").  Returns the moved prompts [(pid, slots)]."""
        if self.peer is None:
            return []
        pids = sorted(pid for pid, p in self.prompts.items()
                      if p.state == SWAPPED and p.location == LOC_PEER)
        fids = sorted(f for f, p in self.prefixes.items() if p.location == LOC_PEER)
        need = sum(len(self.prompts[p].slots) for p in pids) + sum(len(self.prefixes[f].slots) for f in fids)
        if need and (self.host is None or need > len(self.host.free)):
            raise AquaError(E_NOSPACE, "host cannot hold the lender's images")
        moved = self._move([self.prompts[p] for p in pids], LOC_HOST)
        self._move([self.prefixes[f] for f in fids], LOC_HOST)
        self.peer = None
        return list(zip(pids, moved))

    # ---------------------------------------------------------- NEXT-2
    def prefix_store(self, fid: int, src_pid: int, n: int) -> tuple:
        """Persist the first n blocks of a RESIDENT prompt as a cached prefix
        image (Sec. 8: "a new prefill caching API with unique IDs, and
        both CFS and prefill caching share the same swap space"; Sec. 9
        P:895-896).  Copy, not move: the prompt keeps its
        blocks.  Placement as swap_out (R5).  Per j < n, l, kv:
            arena[s_j*U + (2l+kv)*S : +S] = chunk(l, kv, bt[j])
        Errors: fid in use / bad n -> INVAL; src not resident -> STATE;
        no room -> NOSPACE.  Returns (location, slots)."""
        lay = self.lay
        p = self.prompts.get(int(src_pid))
        if int(fid) in self.prefixes:
            raise AquaError(E_INVAL, "prefix id in use")
        if p is None or p.state != RESIDENT:
            raise AquaError(E_STATE, "src not resident")
        if n < 0 or n > len(p.blocks):
            raise AquaError(E_INVAL, "bad block count")
        if self.peer is not None and len(self.peer.free) >= n:
            loc = LOC_PEER
        elif self.host is not None and len(self.host.free) >= n:
            loc = LOC_HOST
        else:
            raise AquaError(E_NOSPACE, "no swap space for the prefix")
        ar = self.arena(loc)
        slots = sorted(ar.free)[:n]
        for s in slots:
            ar.free.remove(s)
        if self.layers is not None and ar.data is not None:
            for b, s in zip(p.blocks[:n], slots):
                for l in range(lay.L):
                    for kv in (0, 1):
                        off = s * lay.U + (2 * l + kv) * lay.S
                        ar.data[off:off + lay.S] = self.chunk(l, kv, b)
        self.prefixes[int(fid)] = Prompt(SWAPPED, [], loc, list(slots))
        return loc, list(slots)

    def prefix_load(self, fid: int, dst_pid: int) -> List[int]:
        """A prefix-cache hit: append n fresh blocks (lowest first, R4) to
        dst_pid (created RESIDENT if new) and copy the cached image into
        them; the image stays for the next hit.  Errors: unknown fid or dst
        swapped -> STATE; pool too small -> NOBLOCKS."""
        lay = self.lay
        f = self.prefixes.get(int(fid))
        if f is None:
            raise AquaError(E_STATE, "unknown prefix")
        p = self.prompts.get(int(dst_pid))
        if p is not None and p.state != RESIDENT:
            raise AquaError(E_STATE, "dst swapped")
        if len(f.slots) > len(self.free):
            raise AquaError(E_NOBLOCKS, "pool exhausted")
        new = self._take_lowest(len(f.slots))
        ar = self.arena(f.location)
        if f.slots and self.layers is not None and ar.data is not None:
            for b, s in zip(new, f.slots):
                for l in range(lay.L):
                    for kv in (0, 1):
                        off = s * lay.U + (2 * l + kv) * lay.S
                        self.chunk(l, kv, b)[:] = ar.data[off:off + lay.S]
        if p is None:
            p = self.prompts[int(dst_pid)] = Prompt(RESIDENT, [], LOC_LOCAL, [])
        p.blocks.extend(new)
        return new

    def prefix_drop(self, fid: int) -> None:
        f = self.prefixes.pop(int(fid), None)
        if f is None:
            raise AquaError(E_STATE, "unknown prefix")
        if f.slots:
            self.arena(f.location).free.update(f.slots)

    # ---------------------------------------------------------------- C-6
    def free_prompt(self, pid: int) -> None:
        """aqua_free: RESIDENT -> blocks back; SWAPPED -> slots back; the
        pid is forgotten ("Freeing allocated tensors")."""
        p = self.prompts.get(int(pid))
        if p is None:
            raise AquaError(E_STATE, "unknown pid")
        if p.state == RESIDENT:
            self.free.update(p.blocks)
        elif p.slots:
            self.arena(p.location).free.update(p.slots)
        del self.prompts[int(pid)]

    def query(self, pid: int):
        """(state, location, n_blocks, ids_or_slots) -- P:855-857 "the
        serving engine can query AquaLib for the tensor location"."""
        p = self.prompts.get(int(pid))
        if p is None:
            raise AquaError(E_STATE, "unknown pid")
        ids = p.blocks if p.state == RESIDENT else p.slots
        return p.state, p.location, len(ids), list(ids)

    # ---------------------------------------------------------- invariants
    def check_invariants(self) -> None:
        """I3 conservation and I4 exclusivity."""
        owned = [b for p in self.prompts.values() if p.state == RESIDENT for b in p.blocks]
        assert len(owned) == len(set(owned)), "block double-owned"
        assert not (set(owned) & self.free), "block both free and owned"
        assert len(self.free) + len(owned) == self.lay.NB, "blocks not conserved"
        for loc in (LOC_PEER, LOC_HOST):
            ar = self.arena(loc)
            if ar is None:
                continue
            used = [s for p in list(self.prompts.values()) + list(self.prefixes.values())
                    if p.state == SWAPPED and p.location == loc for s in p.slots]
            assert len(used) == len(set(used)), "slot double-owned"
            assert not (set(used) & ar.free), "slot both free and owned"
            assert len(ar.free) + len(used) == ar.nslots, "slots not conserved"
