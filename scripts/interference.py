"""NEXT-4 (interference, P:1027-1028 / P:1046-1049): how much does paging slow
an HBM-bound decode running at the same time, and how much paging throughput
is left, as a function of the SMs the swap kernel may use (AQUA_OPT_MAX_CTAS)
and of stream priority.

Decode proxy: one pass over W GB of "weights" (torch reduction, HBM-bound;
16 GB ~ Llama-3-8B bf16 = one decode step's weight read).  Swap: preempt +
resume of the C2 prompt (2 x 4 GiB) on the self-lender.  Prints JSON lines.

    python scripts/interference.py [--weights-gb 16]
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2407_21255_b200 import aqua  # noqa: E402
from workloads import block_permutation  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--weights-gb", type=float, default=16.0)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    L, bs, H, D, NB, nblk = 32, 16, 8, 128, 4096, 2048
    S = bs * H * D * 2
    U = 2 * L * S
    layers = [torch.zeros(2 * NB * S, dtype=torch.uint8, device="cuda") for _ in range(L)]
    arena = torch.empty(nblk * U, dtype=torch.uint8, device="cuda")
    ctx = aqua.Ctx(0, L, bs, H, D, 2, NB, [t.data_ptr() for t in layers])
    ctx.lend(0, arena.data_ptr(), nblk * U)
    perm = block_permutation(NB, NB, seed=2).tolist()
    ctx.adopt_blocks(1, perm[nblk:])
    ctx.adopt_blocks(7, perm[:nblk])
    w = torch.ones(int(args.weights_gb * 1e9) // 8, dtype=torch.int64, device="cuda")
    out = torch.empty((), dtype=torch.int64, device="cuda")

    def timed(fn, stream):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        return a, b

    def decode_once(st):
        with torch.cuda.stream(st):
            torch.sum(w, dim=0, out=out)

    def swap_once(st):
        ctx.swap_out([7], st.cuda_stream)
        ctx.swap_in([7], st.cuda_stream)

    for prio_name, dec_prio, swp_prio in (("equal", 0, 0), ("decode_high", -1, 0)):
        dec = torch.cuda.Stream(priority=dec_prio)
        swp = torch.cuda.Stream(priority=swp_prio)
        for ctas in (0, 74, 32, 16, 8):
            ctx.set_option(aqua.OPT_MAX_CTAS, ctas)
            # alone
            alone_d, alone_s = [], []
            for _ in range(args.reps + 1):
                a, b = timed(lambda: decode_once(dec), dec)
                torch.cuda.synchronize()
                alone_d.append(a.elapsed_time(b))
                a, b = timed(lambda: swap_once(swp), swp)
                torch.cuda.synchronize()
                alone_s.append(a.elapsed_time(b))
            # together: decode steps back to back while one swap pair runs
            tog_d, tog_s = [], []
            for _ in range(args.reps + 1):
                torch.cuda.synchronize()
                sa, sb = timed(lambda: swap_once(swp), swp)
                evs = []
                for _k in range(4):
                    evs.append(timed(lambda: decode_once(dec), dec))
                torch.cuda.synchronize()
                tog_s.append(sa.elapsed_time(sb))
                # decode steps that overlapped the swap window
                tog_d.append(statistics.mean(a.elapsed_time(b) for a, b in evs[:2]))
            d0, s0 = statistics.median(alone_d[1:]), statistics.median(alone_s[1:])
            d1, s1 = statistics.median(tog_d[1:]), statistics.median(tog_s[1:])
            print(json.dumps({"priority": prio_name, "max_ctas": ctas or 148,
                              "decode_alone_ms": round(d0, 3), "decode_with_swap_ms": round(d1, 3),
                              "decode_slowdown": round(d1 / d0, 3),
                              "swap_alone_ms": round(s0, 3), "swap_with_decode_ms": round(s1, 3),
                              "swap_GBps_with_decode": round(2 * nblk * U / s1 / 1e6, 1)}), flush=True)


if __name__ == "__main__":
    main()
