"""Thin ctypes binding of the native CFS scheduler (include/aqua_cfs.h)."""
from __future__ import annotations

import ctypes as C
from typing import List, Tuple

from .aqua import AquaError, lib

POLICY_CFS, POLICY_FCFS = 0, 1
PHASE_PREFILL, PHASE_DECODE = 0, 1

SYMBOLS = ["aqua_trace_run", "aqua_cfs_create", "aqua_cfs_destroy", "aqua_cfs_add", "aqua_cfs_set_state", "aqua_cfs_next",
           "aqua_cfs_commit", "aqua_cfs_partition", "aqua_cfs_set_policy", "aqua_cfs_vclock", "aqua_cfs_advance_to", "aqua_cfs_stats"]


class Config(C.Structure):
    _fields_ = [("policy", C.c_int32), ("batch_tokens", C.c_int32), ("k", C.c_int32),
                ("block_tokens", C.c_int32), ("num_blocks", C.c_int32), ("pad_", C.c_int32),
                ("t_base", C.c_double), ("t_token", C.c_double)]


class Work(C.Structure):
    _fields_ = [("pid", C.c_uint64), ("ctx0", C.c_int32), ("tokens", C.c_int32), ("grow", C.c_int32),
                ("phase", C.c_int32)]


class TraceReq(C.Structure):
    _fields_ = [("pid", C.c_uint64), ("arrival", C.c_double), ("prompt_tokens", C.c_int32),
                ("output_tokens", C.c_int32)]


class TraceOpts(C.Structure):
    _fields_ = [("decode_stream", C.c_void_p), ("swap_stream", C.c_void_p), ("swap_stream2", C.c_void_p),
                ("exchange_pieces", C.c_int32), ("fill", C.c_int32), ("fill_seed", C.c_uint64),
                ("d_mismatches", C.c_void_p)]


class TraceStats(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("swap_out_calls", C.c_int64), ("swap_in_calls", C.c_int64),
                ("blocks_out", C.c_int64), ("blocks_in", C.c_int64), ("vclock", C.c_double)]


_P, _I32, _U64, _VP = C.POINTER, C.c_int32, C.c_uint64, C.c_void_p
for _n, _a in {
    "aqua_cfs_create": [_P(Config), _P(_VP)],
    "aqua_cfs_destroy": [_VP],
    "aqua_cfs_add": [_VP, _U64, C.c_double, _I32, _I32],
    "aqua_cfs_set_state": [_VP, _U64, _I32, _I32, _I32, _I32],
    "aqua_cfs_next": [_VP, _P(_I32), _P(_U64), _P(_I32), _P(_U64), _P(_I32), _P(Work), _P(_I32), _I32],
    "aqua_cfs_commit": [_VP, _P(_U64), _P(_I32), _I32, _P(C.c_double)],
    "aqua_cfs_partition": [_VP, _P(_U64), _P(_I32), _P(_U64), _P(_I32), _P(_I32), _I32],
    "aqua_cfs_vclock": [_VP, _P(C.c_double)],
    "aqua_cfs_set_policy": [_VP, _I32],
    "aqua_cfs_advance_to": [_VP, C.c_double],
    "aqua_cfs_stats": [_VP, _P(_I32), _P(_I32), _P(C.c_int64)],
    "aqua_trace_run": [_VP, _VP, _I32, _P(TraceReq), _P(TraceOpts), _P(TraceStats), _P(C.c_int64), C.c_int64,
                       _P(C.c_int64)],
}.items():
    _f = getattr(lib, _n)
    _f.restype, _f.argtypes = C.c_int, _a


class Scheduler:
    def __init__(self, NB: int, bs: int = 16, b: int = 512, k: int = 8, policy: int = POLICY_CFS,
                 t_base: float = 0.020, t_token: float = 40e-6, cap: int = 1 << 16):
        cfg = Config(policy, b, k, bs, NB, 0, t_base, t_token)
        h = C.c_void_p()
        self._call("aqua_cfs_create", C.byref(cfg), C.byref(h))
        self.h = h
        self.cap = cap
        self._out = (C.c_uint64 * cap)()
        self._in = (C.c_uint64 * cap)()
        self._work = (Work * cap)()
        self._fin = (C.c_uint64 * cap)()
        self._dec = (C.c_uint64 * cap)()
        self._pre = (C.c_uint64 * cap)()
        self._pret = (C.c_int32 * cap)()

    def _call(self, name, *args):
        st = getattr(lib, name)(*args)
        if st != 0:
            raise AquaError(st, name)

    def close(self):
        if getattr(self, "h", None):
            lib.aqua_cfs_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def add(self, pid: int, arrival: float, P: int, O: int) -> None:
        self._call("aqua_cfs_add", self.h, pid, arrival, P, O)

    def set_state(self, pid: int, phase: int, f: int, g: int, ctx: int) -> None:
        self._call("aqua_cfs_set_state", self.h, pid, phase, f, g, ctx)

    def next(self):
        """-> (rescheduled, page_out, page_in, [(pid, ctx0, tokens, grow, phase)])"""
        r, no, ni, nw = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        self._call("aqua_cfs_next", self.h, C.byref(r), self._out, C.byref(no), self._in, C.byref(ni),
                   self._work, C.byref(nw), self.cap)
        work = [(w.pid, w.ctx0, w.tokens, w.grow, w.phase) for w in self._work[:nw.value]]
        return bool(r.value), list(self._out[:no.value]), list(self._in[:ni.value]), work

    def commit(self) -> Tuple[List[int], float]:
        n, v = C.c_int32(), C.c_double()
        self._call("aqua_cfs_commit", self.h, self._fin, C.byref(n), self.cap, C.byref(v))
        return list(self._fin[:n.value]), v.value

    def partition(self):
        nd, npf = C.c_int32(), C.c_int32()
        self._call("aqua_cfs_partition", self.h, self._dec, C.byref(nd), self._pre, self._pret, C.byref(npf),
                   self.cap)
        return list(self._dec[:nd.value]), list(zip(self._pre[:npf.value], self._pret[:npf.value]))

    def set_policy(self, policy: int) -> None:
        self._call("aqua_cfs_set_policy", self.h, policy)

    def vclock(self) -> float:
        v = C.c_double()
        self._call("aqua_cfs_vclock", self.h, C.byref(v))
        return v.value

    def advance_to(self, t: float) -> None:
        self._call("aqua_cfs_advance_to", self.h, t)

    def stats(self):
        a, b, c = C.c_int32(), C.c_int32(), C.c_int64()
        self._call("aqua_cfs_stats", self.h, C.byref(a), C.byref(b), C.byref(c))
        return a.value, b.value, c.value


def decode_log(buf) -> List[tuple]:
    """The native trace log (include/aqua_cfs.h) in the oracle's tuple format."""
    out, i, n = [], 0, len(buf)
    while i < n:
        kind = int(buf[i])
        i += 1
        if kind == 1:
            it, nd = int(buf[i]), int(buf[i + 1])
            D = tuple(int(x) for x in buf[i + 2:i + 2 + nd])
            i += 2 + nd
            npf = int(buf[i])
            PF = tuple((int(buf[i + 1 + 2 * k]), int(buf[i + 2 + 2 * k])) for k in range(npf))
            i += 1 + 2 * npf
            out.append(("plan", it, D, PF))
        elif kind == 2:
            m = int(buf[i])
            pids = tuple(int(x) for x in buf[i + 1:i + 1 + m])
            i += 1 + m
            per = []
            for _ in range(m):
                loc, k = int(buf[i]), int(buf[i + 1])
                per.append((loc, tuple(int(x) for x in buf[i + 2:i + 2 + k])))
                i += 2 + k
            out.append(("swap_out", pids, tuple(per)))
        elif kind == 3:
            m = int(buf[i])
            pids = tuple(int(x) for x in buf[i + 1:i + 1 + m])
            i += 1 + m
            per = []
            for _ in range(m):
                k = int(buf[i])
                per.append(tuple(int(x) for x in buf[i + 1:i + 1 + k]))
                i += 1 + k
            out.append(("swap_in", pids, tuple(per)))
        elif kind == 4:
            pid, k = int(buf[i]), int(buf[i + 1])
            out.append(("alloc", pid, tuple(int(x) for x in buf[i + 2:i + 2 + k])))
            i += 2 + k
        elif kind == 5:
            it, k = int(buf[i]), int(buf[i + 1])
            out.append(("iter", it, tuple((int(buf[i + 2 + 3 * j]), int(buf[i + 3 + 3 * j]), int(buf[i + 4 + 3 * j]))
                                          for j in range(k))))
            i += 2 + 3 * k
        elif kind == 6:
            out.append(("free", int(buf[i])))
            i += 1
        else:
            raise ValueError(f"bad trace record {kind} at {i - 1}")
    return out


def run_trace_native(trace, ctx, sched: Scheduler, *, decode_stream: int = 0, swap_stream: int = 0,
                     swap_stream2: int = 0, exchange_pieces: int = 16, fill_seed=None, d_mismatches: int = 0,
                     record_log: bool = True, log_cap: int = 1 << 22):
    """aqua_trace_run: the whole trace loop in native code.  Returns
    (log in the oracle's format or None, stats dict)."""
    import numpy as np
    reqs = (TraceReq * max(len(trace), 1))(*[TraceReq(int(r), float(a), int(P), int(O)) for r, a, P, O in trace])
    opts = TraceOpts(decode_stream or None, swap_stream or None, swap_stream2 or None, exchange_pieces,
                     1 if fill_seed is not None else 0, fill_seed or 0, d_mismatches or None)
    st = TraceStats()
    n = C.c_int64()
    buf = np.empty(log_cap if record_log else 1, dtype=np.int64)
    rc = lib.aqua_trace_run(ctx.h, sched.h, len(trace), reqs, C.byref(opts), C.byref(st),
                            buf.ctypes.data_as(C.POINTER(C.c_int64)) if record_log else None,
                            log_cap if record_log else 0, C.byref(n))
    if rc != 0:
        raise AquaError(rc, f"aqua_trace_run failed (log needs {n.value} entries)")
    stats = {"iters": st.iterations, "swap_out_calls": st.swap_out_calls, "swap_in_calls": st.swap_in_calls,
             "blocks_out": st.blocks_out, "blocks_in": st.blocks_in, "vclock": st.vclock}
    return (decode_log(buf[:n.value]) if record_log else None), stats
