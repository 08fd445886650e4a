"""Thin ctypes binding of libaqua (include/aqua.h).  Argument marshalling
only: every step of the paging path runs in the C++ library and its sm_100a
kernels.  There is no CPU fallback -- if libaqua.so is missing this module
raises at import time; on a box without a GPU only AQUA_DRYRUN contexts
work.

Functions keep the C names without the ``aqua_`` prefix (``Ctx.swap_out`` ->
``aqua_swap_out``).  Streams are passed as integers (``torch.cuda.Stream
.cuda_stream``; 0 = the legacy default stream), device memory as integer
addresses (``tensor.data_ptr()``).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libaqua.so")

OK, E_INVAL, E_NOBLOCKS, E_NOSPACE, E_STATE, E_CUDA, E_PEER = 0, -1, -2, -3, -4, -5, -6
HOST, DRYRUN, MAPPED = -1, -2, -3
RESIDENT, SWAPPED = 1, 2
LOC_LOCAL, LOC_PEER, LOC_HOST = 0, 1, 2
KERNEL_AUTO, KERNEL_TMA, KERNEL_LDST, BASE_PER_CHUNK, BASE_GATHER_TEMP, KERNEL_CE_HOST = 0, 1, 2, 3, 4, 6   # 5 retired
(OPT_KERNEL, OPT_MAX_CTAS, OPT_TMA_PIECE, OPT_TMA_STAGES, OPT_TIMING, OPT_LDST_VARIANT, OPT_TMA_VARIANT,
 OPT_INLINE_MAX, OPT_TMA_SCHED, OPT_TMA_STATIC_PCT, OPT_RATE_GBPS, OPT_PEER_CTAS,
 OPT_PEER_TEST) = (1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13)
TMA_SCHED_AUTO = 1 << 30

# Every symbol include/aqua.h declares (checked by tests/test_abi.py).
SYMBOLS = [
    "aqua_create", "aqua_destroy", "aqua_lend", "aqua_alloc_blocks", "aqua_adopt_blocks",
    "aqua_swap_out", "aqua_swap_in", "aqua_swap_exchange", "aqua_swap_out_layers", "aqua_swap_in_layers", "aqua_free", "aqua_migrate", "aqua_reclaim", "aqua_prefix_store", "aqua_prefix_load",
    "aqua_prefix_drop", "aqua_prefix_query", "aqua_wait", "aqua_sync", "aqua_ticket_done", "aqua_ticket_elapsed",
    "aqua_query", "aqua_counts", "aqua_arena_base", "aqua_arena_info", "aqua_set_option", "aqua_get_option",
    "aqua_last_descriptors", "aqua_launch_count", "aqua_last_launch", "aqua_ipc_export", "aqua_ipc_import",
    "aqua_ipc_close", "aqua_ipc_alloc", "aqua_ipc_free", "aqua_can_access_peer", "aqua_kv_fill_pattern", "aqua_kv_fill_pattern_batch",
    "aqua_kv_verify_pattern",
    "aqua_strerror", "aqua_last_error", "aqua_version",
]


class AquaError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"aqua status {code}: {msg}")
        self.code = code


class KVLayout(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("block_tokens", C.c_int32), ("num_kv_heads", C.c_int32),
                ("head_dim", C.c_int32), ("elem_bytes", C.c_int32), ("num_blocks", C.c_int32),
                ("layer_base", C.POINTER(C.c_void_p)), ("kv_plane_stride", C.c_int64),
                ("block_stride", C.c_int64)]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2407_21255_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, I32, I64, U64, VP = C.POINTER, C.c_int32, C.c_int64, C.c_uint64, C.c_void_p
    sig = {
        "aqua_create": (C.c_int, [C.c_int, P(KVLayout), P(VP)]),
        "aqua_destroy": (C.c_int, [VP]),
        "aqua_lend": (C.c_int, [VP, C.c_int, VP, U64, P(I32)]),
        # hot calls: pointer arguments as raw addresses (VP) of per-Ctx scratch buffers
        "aqua_alloc_blocks": (C.c_int, [VP, U64, I32, VP, VP]),
        "aqua_adopt_blocks": (C.c_int, [VP, U64, I32, P(I32), VP]),
        "aqua_swap_out": (C.c_int, [VP, I32, VP, VP, VP]),
        "aqua_swap_in": (C.c_int, [VP, I32, VP, VP, VP, I64, VP, VP]),
        "aqua_swap_exchange": (C.c_int, [VP, I32, VP, I32, VP, VP, VP, I32, VP, I64, VP, VP, VP]),
        "aqua_swap_out_layers": (C.c_int, [VP, I32, P(U64), VP, I32, P(U64)]),
        "aqua_swap_in_layers": (C.c_int, [VP, I32, P(U64), VP, I32, P(I32), I64, P(I32), P(U64)]),
        "aqua_free": (C.c_int, [VP, U64, VP]),
        "aqua_migrate": (C.c_int, [VP, I32, P(U64), I32, VP, P(U64)]),
        "aqua_reclaim": (C.c_int, [VP, VP, P(U64)]),
        "aqua_prefix_store": (C.c_int, [VP, U64, U64, I32, VP, P(U64)]),
        "aqua_prefix_load": (C.c_int, [VP, U64, U64, VP, P(I32), I32, P(U64)]),
        "aqua_prefix_drop": (C.c_int, [VP, U64]),
        "aqua_prefix_query": (C.c_int, [VP, U64, P(I32), P(I32), P(I32), I32]),
        "aqua_wait": (C.c_int, [VP, U64, VP]),
        "aqua_sync": (C.c_int, [VP, U64]),
        "aqua_ticket_done": (C.c_int, [VP, U64, VP]),
        "aqua_ticket_elapsed": (C.c_int, [VP, U64, P(C.c_float)]),
        "aqua_query": (C.c_int, [VP, U64, P(I32), P(I32), P(I32), P(I32), I32]),
        "aqua_counts": (C.c_int, [VP, P(I32), P(I32), P(I32)]),
        "aqua_arena_base": (C.c_int, [VP, I32, P(VP), P(I32)]),
        "aqua_arena_info": (C.c_int, [VP, I32, P(I32), P(I32), P(I32), P(I32)]),
        "aqua_set_option": (C.c_int, [VP, I32, I64]),
        "aqua_get_option": (C.c_int, [VP, I32, P(I64)]),
        "aqua_last_descriptors": (C.c_int, [VP, P(I32), P(I32), P(I32), I64, P(I64)]),
        "aqua_launch_count": (C.c_int, [VP, P(U64)]),
        "aqua_last_launch": (C.c_int, [VP, P(I32), P(I32), P(I32), P(I32), P(I32), P(I64), P(I64)]),
        "aqua_ipc_export": (C.c_int, [VP, P(C.c_uint8)]),
        "aqua_ipc_import": (C.c_int, [C.c_int, P(C.c_uint8), P(VP)]),
        "aqua_ipc_close": (C.c_int, [C.c_int, VP]),
        "aqua_ipc_alloc": (C.c_int, [C.c_int, U64, P(VP)]),
        "aqua_ipc_free": (C.c_int, [C.c_int, VP]),
        "aqua_can_access_peer": (C.c_int, [C.c_int, C.c_int, P(I32)]),
        "aqua_kv_fill_pattern": (C.c_int, [VP, U64, I32, I32, U64, VP]),
        "aqua_kv_verify_pattern": (C.c_int, [VP, U64, I32, U64, VP, VP]),
        "aqua_kv_fill_pattern_batch": (C.c_int, [VP, I32, P(U64), P(I32), P(I32), U64, VP]),
        "aqua_strerror": (C.c_char_p, [C.c_int]),
        "aqua_last_error": (C.c_char_p, [VP]),
        "aqua_version": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


lib = _load()


def _i32p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _u64p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def _check(st: int, ctx=None):
    if st != OK:
        msg = lib.aqua_last_error(ctx).decode() if ctx is not None else lib.aqua_last_error(None).decode()
        raise AquaError(st, msg or lib.aqua_strerror(st).decode())


class Ctx:
    """One borrower context (aqua_ctx*).  ``layer_ptrs`` are the L device
    addresses of the per-layer KV tensors (caller-owned)."""

    def __init__(self, device: int, L: int, bs: int, H: int, D: int, e: int, NB: int,
                 layer_ptrs: Sequence[int], kv_plane_stride: int = 0, block_stride: int = 0):
        self._ptrs = (C.c_void_p * L)(*[int(p) for p in layer_ptrs])
        lay = KVLayout(L, bs, H, D, e, NB, C.cast(self._ptrs, C.POINTER(C.c_void_p)),
                       kv_plane_stride, block_stride)
        h = C.c_void_p()
        _check(lib.aqua_create(device, C.byref(lay), C.byref(h)))
        self.h = h
        self.L, self.bs, self.H, self.D, self.e, self.NB = L, bs, H, D, e, NB
        self.S = bs * H * D * e
        self.U = 2 * L * self.S
        # Scratch buffers of the hot calls, allocated once with their
        # addresses cached: numpy's .ctypes costs microseconds per call,
        # several times the library's own cost of a small swap
        # (profiles/r02_host_cost.jsonl).  A Ctx is not reentrant.
        self._pid = np.empty(64, np.uint64)
        self._pid_a = self._pid.ctypes.data
        self._pid2 = np.empty(64, np.uint64)
        self._pid2_a = self._pid2.ctypes.data
        self._cnt = np.empty(64, np.int32)
        self._cnt_a = self._cnt.ctypes.data
        self._ids = np.empty(max(NB, 1), np.int32)     # no call returns more than NB block ids
        self._ids_a = self._ids.ctypes.data
        self._tk = (C.c_uint64 * 2)()
        self._tk_a = C.addressof(self._tk)
        self._d32 = C.c_int32()
        self._d32_a = C.addressof(self._d32)

    def close(self):
        if self.h:
            lib.aqua_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _c(self, st):
        _check(st, self.h)

    def lend(self, lender_device: int, base: int = 0, nbytes: int = 0) -> int:
        n = C.c_int32()
        self._c(lib.aqua_lend(self.h, lender_device, C.c_void_p(base or None), nbytes, C.byref(n)))
        return n.value

    def _pids_arg(self, pids, second: bool = False) -> int:
        """Copies pids into a scratch buffer; returns its address."""
        n = len(pids)
        buf = self._pid2 if second else self._pid
        if n > len(buf):
            buf = np.empty(2 * n, np.uint64)
            if second:
                self._pid2, self._pid2_a = buf, buf.ctypes.data
            else:
                self._pid, self._pid_a = buf, buf.ctypes.data
        if n == 1:
            buf[0] = pids[0]
        elif n:
            buf[:n] = pids
        return self._pid2_a if second else self._pid_a

    def _counts_arg(self, n: int) -> int:
        if n > len(self._cnt):
            self._cnt = np.empty(2 * n, np.int32)
            self._cnt_a = self._cnt.ctypes.data
        return self._cnt_a

    def _tables(self, n: int, as_arrays: bool = False):
        """The new block tables of an n-prompt swap-in from the scratch buffers
        (lists of ints, or int32 numpy copies with as_arrays)."""
        conv = np.ndarray.copy if as_arrays else np.ndarray.tolist
        if n == 1:
            return [conv(self._ids[:int(self._cnt[0])])]
        ids, cnt = self._ids, self._cnt[:n].tolist()
        out, k = [], 0
        for c in cnt:
            out.append(conv(ids[k:k + c]))
            k += c
        return out

    def alloc_blocks(self, pid: int, n: int, stream: int = 0) -> List[int]:
        if 0 <= n <= len(self._ids):
            st = lib.aqua_alloc_blocks(self.h, pid, n, stream or None, self._ids_a)
            if st:
                _check(st, self.h)
            return self._ids[:n].tolist()
        out = np.empty(max(n, 1), np.int32)
        self._c(lib.aqua_alloc_blocks(self.h, pid, n, stream or None, out.ctypes.data))
        return out[:n].tolist()

    def adopt_blocks(self, pid: int, ids: Sequence[int], stream: int = 0) -> None:
        a = np.ascontiguousarray(ids, dtype=np.int32)
        self._c(lib.aqua_adopt_blocks(self.h, pid, len(a), _i32p(a), C.c_void_p(stream or None)))

    def swap_out(self, pids: Sequence[int], stream: int = 0) -> int:
        st = lib.aqua_swap_out(self.h, len(pids), self._pids_arg(pids), stream or None, self._tk_a)
        if st:
            _check(st, self.h)
        return self._tk[0]

    def _cap(self, pids) -> int:
        """Capacity for the new block ids of `pids` (0 for unknown pids: the
        C call itself reports the error, in its own order)."""
        n = 0
        st, loc, k = C.c_int32(), C.c_int32(), C.c_int32()
        for p in pids:
            if lib.aqua_query(self.h, int(p), C.byref(st), C.byref(loc), C.byref(k), None, 0) == OK:
                n += k.value
        return n

    def swap_in(self, pids: Sequence[int], stream: int = 0, cap: int = -1,
                as_arrays: bool = False) -> Tuple[list, int]:
        """-> (the new block table of each pid -- a list of ints, or an int32
        numpy array with as_arrays, which skips the per-id Python objects --,
        the ticket)"""
        n = len(pids)
        if cap < 0:
            # the scratch holds NB ids, the most a pool can hand out; a call
            # needing more gets the exact capacity so that the library reports
            # its own error (pool exhausted) rather than "out_ids too small"
            st = lib.aqua_swap_in(self.h, n, self._pids_arg(pids), stream or None, self._ids_a, len(self._ids),
                                  self._counts_arg(n), self._tk_a)
            if st == OK:
                return self._tables(n, as_arrays), self._tk[0]
            if st != E_INVAL or b"out_ids too small" not in (lib.aqua_last_error(self.h) or b""):
                _check(st, self.h)
            cap = self._cap(pids)
        ids = np.empty(max(cap, 1), np.int32)
        counts = np.empty(max(n, 1), np.int32)
        self._c(lib.aqua_swap_in(self.h, n, self._pids_arg(pids), stream or None, ids.ctypes.data, cap,
                                 counts.ctypes.data, self._tk_a))
        out, k = [], 0
        for i in range(n):
            seg = ids[k:k + counts[i]]
            out.append(seg.copy() if as_arrays else seg.tolist())
            k += counts[i]
        return out, self._tk[0]

    def swap_exchange(self, out_pids: Sequence[int], in_pids: Sequence[int], out_stream: int = 0,
                      in_stream: int = 0, pieces: int = 16):
        """-> (new block tables of in_pids, out_ticket, in_ticket)"""
        na, nb = len(out_pids), len(in_pids)
        cap = self._cap(in_pids)
        ids = self._ids if cap <= len(self._ids) else np.empty(cap, np.int32)
        a_addr = self._pids_arg(out_pids)
        b_addr = self._pids_arg(in_pids, second=True)
        self._c(lib.aqua_swap_exchange(self.h, na, a_addr, nb, b_addr, out_stream or None, in_stream or None, pieces,
                                       ids.ctypes.data if ids is not self._ids else self._ids_a, max(cap, 0),
                                       self._counts_arg(nb), self._tk_a, self._tk_a + 8))
        out, k = [], 0
        for c in self._cnt[:nb].tolist():
            out.append(ids[k:k + c].tolist())
            k += c
        return out, self._tk[0], self._tk[1]

    def swap_out_layers(self, pids: Sequence[int], layer_group: int, stream: int = 0) -> List[int]:
        a = np.ascontiguousarray(pids, dtype=np.uint64)
        ng = -(-self.L // layer_group) if layer_group > 0 else 1
        t = np.zeros(max(ng, 1), np.uint64)
        self._c(lib.aqua_swap_out_layers(self.h, len(a), _u64p(a), C.c_void_p(stream or None), layer_group,
                                         _u64p(t)))
        return [int(x) for x in t[:ng]]

    def swap_in_layers(self, pids: Sequence[int], layer_group: int, stream: int = 0):
        a = np.ascontiguousarray(pids, dtype=np.uint64)
        cap = self._cap(a)
        ids = np.empty(max(cap, 1), np.int32)
        counts = np.empty(max(len(a), 1), np.int32)
        ng = -(-self.L // layer_group) if layer_group > 0 else 1
        t = np.zeros(max(ng, 1), np.uint64)
        self._c(lib.aqua_swap_in_layers(self.h, len(a), _u64p(a), C.c_void_p(stream or None), layer_group,
                                        _i32p(ids), cap, _i32p(counts), _u64p(t)))
        out, k = [], 0
        for i in range(len(a)):
            out.append(ids[k:k + counts[i]].tolist())
            k += counts[i]
        return out, [int(x) for x in t[:ng]]

    def free(self, pid: int, stream: int = 0) -> None:
        st = lib.aqua_free(self.h, pid, stream or None)
        if st:
            _check(st, self.h)

    def migrate(self, pids: Sequence[int], dst_loc: int, stream: int = 0) -> int:
        a = np.ascontiguousarray(pids, dtype=np.uint64)
        t = C.c_uint64()
        self._c(lib.aqua_migrate(self.h, len(a), _u64p(a), dst_loc, C.c_void_p(stream or None), C.byref(t)))
        return t.value

    def reclaim(self, stream: int = 0) -> int:
        t = C.c_uint64()
        self._c(lib.aqua_reclaim(self.h, C.c_void_p(stream or None), C.byref(t)))
        return t.value

    def prefix_store(self, fid: int, src_pid: int, n: int, stream: int = 0) -> int:
        t = C.c_uint64()
        self._c(lib.aqua_prefix_store(self.h, fid, src_pid, n, C.c_void_p(stream or None), C.byref(t)))
        return t.value

    def prefix_query(self, fid: int):
        loc, n = C.c_int32(), C.c_int32()
        self._c(lib.aqua_prefix_query(self.h, fid, C.byref(loc), C.byref(n), None, 0))
        sl = np.empty(max(n.value, 1), np.int32)
        self._c(lib.aqua_prefix_query(self.h, fid, None, None, _i32p(sl), n.value))
        return loc.value, sl[:n.value].tolist()

    def prefix_load(self, fid: int, dst_pid: int, stream: int = 0) -> Tuple[List[int], int]:
        n = self.prefix_query(fid)[1]
        ids = np.empty(max(len(n), 1), np.int32)
        t = C.c_uint64()
        self._c(lib.aqua_prefix_load(self.h, fid, dst_pid, C.c_void_p(stream or None), _i32p(ids), len(n),
                                     C.byref(t)))
        return ids[:len(n)].tolist(), t.value

    def prefix_drop(self, fid: int) -> None:
        self._c(lib.aqua_prefix_drop(self.h, fid))

    def wait(self, ticket: int, stream: int = 0) -> None:
        st = lib.aqua_wait(self.h, ticket, stream or None)
        if st:
            _check(st, self.h)

    def sync(self, ticket: int) -> None:
        self._c(lib.aqua_sync(self.h, ticket))

    def ticket_done(self, ticket: int) -> bool:
        self._c(lib.aqua_ticket_done(self.h, ticket, self._d32_a))
        return bool(self._d32.value)

    def ticket_elapsed(self, ticket: int) -> float:
        v = C.c_float()
        self._c(lib.aqua_ticket_elapsed(self.h, ticket, C.byref(v)))
        return v.value

    def query(self, pid: int, with_ids: bool = False):
        st, loc, n = C.c_int32(), C.c_int32(), C.c_int32()
        self._c(lib.aqua_query(self.h, pid, C.byref(st), C.byref(loc), C.byref(n), None, 0))
        if not with_ids:
            return st.value, loc.value, n.value
        ids = np.empty(max(n.value, 1), np.int32)
        self._c(lib.aqua_query(self.h, pid, None, None, None, _i32p(ids), n.value))
        return st.value, loc.value, n.value, ids[:n.value].tolist()

    def counts(self) -> Tuple[int, int, int]:
        a, b, c = C.c_int32(), C.c_int32(), C.c_int32()
        self._c(lib.aqua_counts(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def arena_base(self, loc: int) -> Tuple[int, int]:
        p, n = C.c_void_p(), C.c_int32()
        self._c(lib.aqua_arena_base(self.h, loc, C.byref(p), C.byref(n)))
        return p.value or 0, n.value

    def arena_info(self, which: int) -> dict:
        """aqua_arena_info: which = LOC_PEER (the GPU lender) or LOC_HOST."""
        d, pe, pr, n = (C.c_int32() for _ in range(4))
        self._c(lib.aqua_arena_info(self.h, which, C.byref(d), C.byref(pe), C.byref(pr), C.byref(n)))
        return {"device": d.value, "peer": bool(pe.value), "probe": pr.value, "nslots": n.value}

    def set_option(self, opt: int, value: int) -> None:
        self._c(lib.aqua_set_option(self.h, opt, value))

    def get_option(self, opt: int) -> int:
        v = C.c_int64()
        self._c(lib.aqua_get_option(self.h, opt, C.byref(v)))
        return v.value

    def last_descriptors(self):
        n = C.c_int64()
        self._c(lib.aqua_last_descriptors(self.h, None, None, None, 0, C.byref(n)))
        b = np.empty(max(n.value, 1), np.int32)
        s = np.empty_like(b)
        l = np.empty_like(b)
        self._c(lib.aqua_last_descriptors(self.h, _i32p(b), _i32p(s), _i32p(l), n.value, C.byref(n)))
        k = n.value
        return b[:k].tolist(), s[:k].tolist(), l[:k].tolist()

    def launch_count(self) -> int:
        v = C.c_uint64()
        self._c(lib.aqua_launch_count(self.h, C.byref(v)))
        return v.value

    def last_launch(self) -> dict:
        """Shape of the most recent swap / migrate kernel launch (aqua_last_launch)."""
        g, t, st, en, va = (C.c_int32() for _ in range(5))
        b, il = C.c_int64(), C.c_int64()
        self._c(lib.aqua_last_launch(self.h, C.byref(g), C.byref(t), C.byref(st), C.byref(en), C.byref(va),
                                     C.byref(b), C.byref(il)))
        return {"ctas": g.value, "threads_per_cta": t.value, "stages": st.value,
                "engine": {KERNEL_TMA: "tma", KERNEL_LDST: "ldst"}.get(en.value, en.value), "variant": va.value,
                "schedule": f"claimed batches of {b.value} items" if b.value > 0 else "static ranges",
                "inline_descriptors": il.value}

    def kv_fill_pattern(self, pid: int, t0: int, t1: int, seed: int, stream: int = 0) -> None:
        self._c(lib.aqua_kv_fill_pattern(self.h, pid, t0, t1, seed, C.c_void_p(stream or None)))

    def kv_fill_pattern_batch(self, pids: Sequence[int], t0s: Sequence[int], t1s: Sequence[int], seed: int,
                              stream: int = 0) -> None:
        a = np.ascontiguousarray(pids, dtype=np.uint64)
        b = np.ascontiguousarray(t0s, dtype=np.int32)
        e = np.ascontiguousarray(t1s, dtype=np.int32)
        self._c(lib.aqua_kv_fill_pattern_batch(self.h, len(a), _u64p(a), _i32p(b), _i32p(e), seed,
                                               C.c_void_p(stream or None)))

    def kv_verify_pattern(self, pid: int, ntok: int, seed: int, d_counter: int, stream: int = 0) -> None:
        self._c(lib.aqua_kv_verify_pattern(self.h, pid, ntok, seed, C.c_void_p(stream or None),
                                           C.c_void_p(d_counter)))


def ipc_export(dev_ptr: int) -> bytes:
    h = (C.c_uint8 * 64)()
    _check(lib.aqua_ipc_export(C.c_void_p(dev_ptr), h))
    return bytes(h)


def ipc_import(device: int, handle: bytes) -> int:
    h = (C.c_uint8 * 64)(*handle)
    p = C.c_void_p()
    _check(lib.aqua_ipc_import(device, h, C.byref(p)))
    return p.value


def ipc_close(device: int, ptr: int) -> None:
    _check(lib.aqua_ipc_close(device, C.c_void_p(ptr)))


def ipc_alloc(device: int, nbytes: int) -> int:
    p = C.c_void_p()
    _check(lib.aqua_ipc_alloc(device, nbytes, C.byref(p)))
    return p.value


def ipc_free(device: int, ptr: int) -> None:
    _check(lib.aqua_ipc_free(device, C.c_void_p(ptr)))


def can_access_peer(device: int, peer: int) -> bool:
    v = C.c_int32()
    _check(lib.aqua_can_access_peer(device, peer, C.byref(v)))
    return bool(v.value)


def version() -> str:
    return lib.aqua_version().decode()
