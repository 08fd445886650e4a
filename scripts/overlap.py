"""A8 (paging overlaps decode; north_star "paging overlaps decode"):
does a swap on its own stream run concurrently with an HBM-bound decode?

    python scripts/overlap.py [--weights-gb 16] [--steps 40]

Decode proxy: `steps` decode iterations, each one pass over W GB of "weights"
(torch reduction, HBM-bound) on the decode stream.  Paging: preempt + resume
of prompts that the decode does NOT touch (the C2 prompt, 2 x 4 GiB), on a
swap stream -- the case the tickets allow to overlap (a prompt being paged
out is not in the next batch).  Three placements of the images:

  host      pinned DRAM over PCIe through the copy engines (AUTO: CE_HOST):
            the copy engines hold no SMs and the PCIe traffic is ~1 % of HBM
            bandwidth, so overlapped ~= max(decode, paging);
  host_sm   the same through the zero-copy TMA kernel (8 SMs);
  self      the same GPU's HBM (self-lender): both sides are HBM-bound, so
            overlap cannot beat the sum of the HBM traffic (what round 1's C3
            runs measured: separate streams = one stream);
  mixed     half the blocks (one prompt) fill a self-lender arena exactly,
            the other prompt falls back to pinned DRAM (R5), both paged in
            ONE call: AUTO splits it (TMA kernel for the lender images, copy
            engines for the host ones);
  mixed_tma the same call as one fused TMA launch (AQUA_KERNEL_TMA; AUTO
            before the split), which holds its SMs for the PCIe time.

For each: decode alone, paging alone, both serialised on one stream, and both
on separate streams; prints one JSON line per placement with the overlap
gain = serial / concurrent and the fraction of the shorter side hidden.

--decode gemm swaps the decode proxy for a tensor-core-bound one (bf16
GEMMs, the weight-multiply part of a large-batch decode step): then the two
sides compete for SMs, not HBM, and --caps (AQUA_OPT_MAX_CTAS values for the
self-lender swap) trades paging speed against the SMs left to the GEMMs --
the CTA-cap mitigation of NEXT-4.
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2407_21255_b200 import aqua  # noqa: E402
from workloads import block_permutation  # noqa: E402

L, bs, H, D, NB = 32, 16, 8, 128, 4096
S = bs * H * D * 2
U = 2 * L * S


def _ctas(ctx):
    try:
        return ctx.last_launch()["ctas"]
    except aqua.AquaError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--weights-gb", type=float, default=16.0)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--nblk", type=int, default=2048)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--decode", choices=["hbm", "gemm"], default="hbm")
    ap.add_argument("--gemm", type=int, default=8192, help="M = N = K of one decode-step GEMM (bf16)")
    ap.add_argument("--images", default="host,host_sm,self")
    ap.add_argument("--caps", default="0", help="comma-separated SM caps for the self-lender swap (0 = all SMs)")
    args = ap.parse_args()
    nblk = args.nblk
    layers = [torch.zeros(2 * NB * S, dtype=torch.uint8, device="cuda") for _ in range(L)]
    if args.decode == "hbm":
        w = torch.ones(int(args.weights_gb * 1e9) // 8, dtype=torch.int64, device="cuda")
        out = torch.empty((), dtype=torch.int64, device="cuda")
    else:
        g = args.gemm
        ga = torch.randn(g, g, device="cuda", dtype=torch.bfloat16)
        gb = torch.randn(g, g, device="cuda", dtype=torch.bfloat16)
        gc = torch.empty(g, g, device="cuda", dtype=torch.bfloat16)
    dec = torch.cuda.Stream()
    swp = torch.cuda.Stream()
    perm = block_permutation(NB, NB, seed=2).tolist()

    runs = []
    for where in args.images.split(","):
        for cap in ([int(c) for c in args.caps.split(",")] if where == "self" else [0]):
            runs.append((where, cap))
    for where, cap in runs:
        ctx = aqua.Ctx(0, L, bs, H, D, 2, NB, [t.data_ptr() for t in layers])
        if cap:
            ctx.set_option(aqua.OPT_MAX_CTAS, cap)
        arena = None
        pids = [7]
        if where in ("mixed", "mixed_tma"):
            half = nblk // 2
            arena = torch.empty(half * U, dtype=torch.uint8, device="cuda")
            ctx.lend(0, arena.data_ptr(), half * U)
            ctx.lend(aqua.HOST, 0, (nblk - half) * U)
            if where == "mixed_tma":
                ctx.set_option(aqua.OPT_KERNEL, aqua.KERNEL_TMA)
            pids = [7, 8]
        elif where == "self":
            arena = torch.empty(nblk * U, dtype=torch.uint8, device="cuda")
            ctx.lend(0, arena.data_ptr(), nblk * U)
        else:
            ctx.lend(aqua.HOST, 0, nblk * U)
            if where == "host_sm":
                ctx.set_option(aqua.OPT_KERNEL, aqua.KERNEL_TMA)
        ctx.adopt_blocks(1, perm[nblk:])
        if len(pids) == 1:
            ctx.adopt_blocks(7, perm[:nblk])
        else:
            ctx.adopt_blocks(7, perm[:nblk // 2])
            ctx.adopt_blocks(8, perm[nblk // 2:nblk])
            ctx.swap_out(pids)                   # placement check: lender exactly full, then host (R5)
            assert (ctx.query(7)[1], ctx.query(8)[1]) == (aqua.LOC_PEER, aqua.LOC_HOST)
            ctx.swap_in(pids)
            torch.cuda.synchronize()

        def decode(st, n):
            with torch.cuda.stream(st):
                for _ in range(n):
                    if args.decode == "hbm":
                        torch.sum(w, dim=0, out=out)
                    else:
                        torch.matmul(ga, gb, out=gc)

        def page(st):
            ctx.swap_out(pids, st.cuda_stream)
            ctx.swap_in(pids, st.cuda_stream)

        def timed(fn):
            best = None
            for _ in range(args.reps):
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(torch.cuda.current_stream())
                fn()
                for st in (dec, swp):
                    torch.cuda.current_stream().wait_stream(st)
                b.record(torch.cuda.current_stream())
                torch.cuda.synchronize()
                ms = a.elapsed_time(b)
                best = ms if best is None else min(best, ms)
            return best

        page(swp)
        decode(dec, 2)
        torch.cuda.synchronize()
        t_page = timed(lambda: page(swp))
        # enough decode steps to span the paging time (at least args.steps)
        t_step = timed(lambda: decode(dec, 1))
        n = max(args.steps, int(t_page / t_step) + 1)
        t_dec = timed(lambda: decode(dec, n))

        def serial():
            for st in (dec, swp):
                st.wait_stream(torch.cuda.current_stream())
            decode(dec, n)
            swp.wait_stream(dec)
            page(swp)

        def concurrent():
            for st in (dec, swp):
                st.wait_stream(torch.cuda.current_stream())
            page(swp)
            decode(dec, n)

        t_ser = timed(serial)
        t_con = timed(concurrent)
        hidden = (t_ser - t_con) / min(t_dec, t_page) if min(t_dec, t_page) > 0 else 0.0
        extra = {}
        if args.decode == "gemm":
            extra["gemm_TFLOPs"] = round(2 * args.gemm ** 3 * n / (t_dec / 1e3) / 1e12, 1)
        print(json.dumps({"images": where, "decode": args.decode, "swap_sm_cap": cap,
                          "swap_ctas": _ctas(ctx), **extra,
                          "decode_steps": n, "decode_ms": round(t_dec, 3),
                          "paging_ms": round(t_page, 3), "paging_GBps": round(2 * nblk * U / t_page / 1e6, 1),
                          "serial_ms": round(t_ser, 3), "concurrent_ms": round(t_con, 3),
                          "overlap_gain": round(t_ser / t_con, 3),
                          "hidden_fraction_of_shorter": round(hidden, 3)}), flush=True)
        ctx.close()
        del arena
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
