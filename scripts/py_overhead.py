"""Where the Python binding's per-call time goes on a GPU box: a 1-block
swap_out / swap_in pair through (a) Ctx methods, (b) the raw ctypes calls
with cached arguments, (c) the same through ctypes.PyDLL (GIL held), and the
cost of reading torch's Stream.cuda_stream.  Prints one JSON line."""
import ctypes as C
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_21255_b200 import aqua  # noqa: E402


def med(f, reps=3000):
    ts = []
    for i in range(reps):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
        if i % 16 == 15:
            torch.cuda.synchronize()
    return round(1e6 * statistics.median(ts[reps // 10:]), 2)


def main():
    L, bs, H, D = 32, 16, 8, 128
    S = bs * H * D * 2
    NB = 64
    layers = [torch.empty(2 * NB * S, dtype=torch.uint8, device="cuda") for _ in range(L)]
    arena = torch.empty(NB * 2 * L * S, dtype=torch.uint8, device="cuda")
    ctx = aqua.Ctx(0, L, bs, H, D, 2, NB, [t.data_ptr() for t in layers])
    ctx.lend(aqua.MAPPED, arena.data_ptr(), arena.numel())
    ctx.alloc_blocks(7, 1)
    s = torch.cuda.Stream()
    sp = s.cuda_stream
    out = {}

    def pair_methods():
        ctx.swap_out([7], sp)
        ctx.swap_in([7], sp)
    out["methods_pair_us"] = med(pair_methods)

    def pair_methods_stream_attr():
        ctx.swap_out([7], s.cuda_stream)
        ctx.swap_in([7], s.cuda_stream)
    out["methods_pair_stream_attr_us"] = med(pair_methods_stream_attr)
    out["stream_attr_us"] = med(lambda: s.cuda_stream)

    lib = aqua.lib
    a = ctx._pids_arg([7])

    def pair_raw():
        lib.aqua_swap_out(ctx.h, 1, a, sp, ctx._tk_a)
        lib.aqua_swap_in(ctx.h, 1, a, sp, ctx._ids_a, NB, ctx._cnt_a, ctx._tk_a)
    out["raw_pair_us"] = med(pair_raw)

    plib = C.PyDLL(aqua.LIB_PATH)
    for name in ("aqua_swap_out", "aqua_swap_in"):
        getattr(plib, name).restype = getattr(lib, name).restype
        getattr(plib, name).argtypes = getattr(lib, name).argtypes

    def pair_pydll():
        plib.aqua_swap_out(ctx.h, 1, a, sp, ctx._tk_a)
        plib.aqua_swap_in(ctx.h, 1, a, sp, ctx._ids_a, NB, ctx._cnt_a, ctx._tk_a)
    out["pydll_pair_us"] = med(pair_pydll)
    out["noop_ctypes_us"] = med(lambda: lib.aqua_version())
    torch.cuda.synchronize()
    ctx.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
