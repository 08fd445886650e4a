"""Peer-lender swap bandwidth over NVLink, one process driving two GPUs
(SURVEY 8(d) C5 / north_star: KV swap GB/s per GPU pair vs 900 GB/s).

    python scripts/nvlink_peer.py [--borrower 0] [--lender 1] [--config c2|c4]
        [--ctas 8,16,24,32,48,64,0] [--bidir] [--steps 10] [--warmup 3]

The borrower's pool holds the config's prompts (fragmented block tables,
closed-form KV pattern); the lender arena is a cudaMalloc on the other GPU,
lent with aqua_lend(lender_device) (P2P enabled by the library, lend-time
probe).  For every peer CTA cap (AQUA_OPT_PEER_CTAS; 0 = all SMs) it times
swap_out (borrower HBM -> lender HBM over NVLink) and swap_in (pull back)
with CUDA events on the swap stream and prints one JSON line per cap:
GB/s per direction, fraction of 900 (nominal) and 770 (measured peer copy),
and the pattern verify of the resumed prompts.  --bidir also runs the
mirror pair (the lender GPU borrowing from the borrower GPU) concurrently,
so both link directions carry swaps (configs[4] "bidirectional").
`--lender 0` on a one-GPU box runs the same code against the borrower's own
HBM (a smoke test of the script; the cap then does not apply: not a peer).

This calibrates the peer CTA cap (the minimum SMs that
carry the link) and is the command the NVLink ncu recipe wraps
(scripts/gpu_runs/r02_nvlink_ncu.sh: --replay-mode application with
nvltx__/nvlrx__bytes_data_user).  On a one-GPU box it prints a skip line.
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

CONFIGS = {"c2": dict(L=32, H=8, NB=4096, nprompts=1, bpp=2048),
           "c4": dict(L=80, H=2, NB=8192, nprompts=32, bpp=128)}
SEED = 1234


class Side:
    """One borrower device paging into one lender device."""

    def __init__(self, bdev, ldev, cfg):
        self.bdev, self.ldev = bdev, ldev
        L, H, NB = cfg["L"], cfg["H"], cfg["NB"]
        self.S = 16 * H * 128 * 2
        self.U = 2 * L * self.S
        self.nblk = cfg["nprompts"] * cfg["bpp"]
        self.pids = list(range(100, 100 + cfg["nprompts"]))
        self.bpp = cfg["bpp"]
        dev = torch.device("cuda", bdev)
        self.layers = [torch.empty(2 * NB * self.S, dtype=torch.uint8, device=dev) for _ in range(L)]
        self.arena = torch.empty(self.nblk * self.U, dtype=torch.uint8, device=torch.device("cuda", ldev))
        self.ctx = aqua.Ctx(bdev, L, 16, H, 128, 2, NB, [t.data_ptr() for t in self.layers])
        self.ctx.lend(ldev, self.arena.data_ptr(), self.nblk * self.U)
        self.info = self.ctx.arena_info(aqua.LOC_PEER)
        perm = block_permutation(NB, NB, seed=2).tolist()
        self.ctx.adopt_blocks(1, perm[self.nblk:])
        for i, pid in enumerate(self.pids):
            self.ctx.adopt_blocks(pid, perm[i * self.bpp:(i + 1) * self.bpp])
            self.ctx.kv_fill_pattern(pid, 0, self.bpp * 16, SEED)
        with torch.cuda.device(bdev):
            self.stream = torch.cuda.Stream()
        torch.cuda.synchronize(bdev)

    def enqueue(self, k, evs):
        sw = self.stream.cuda_stream
        for i in range(k):
            if evs is not None:
                evs[i][0].record(self.stream)
            self.ctx.swap_out(self.pids, sw)
            if evs is not None:
                evs[i][1].record(self.stream)
            self.ctx.swap_in(self.pids, sw)
            if evs is not None:
                evs[i][2].record(self.stream)

    def events(self, k):
        with torch.cuda.device(self.bdev):
            return [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(k)]

    def verify(self):
        cnt = torch.zeros(1, dtype=torch.int64, device=torch.device("cuda", self.bdev))
        for pid in self.pids:
            self.ctx.kv_verify_pattern(pid, self.bpp * 16, SEED, cnt.data_ptr())
        torch.cuda.synchronize(self.bdev)
        return int(cnt.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--borrower", type=int, default=0)
    ap.add_argument("--lender", type=int, default=1)
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--ctas", default="8,16,24,32,48,64,0")
    ap.add_argument("--bidir", action="store_true")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    if max(args.borrower, args.lender) >= torch.cuda.device_count():
        print(json.dumps({"skipped": "needs 2 GPUs (peer lender over NVLink)",
                          "devices": torch.cuda.device_count()}))
        return
    cfg = CONFIGS[args.config]
    sides = [Side(args.borrower, args.lender, cfg)]
    if args.bidir:
        sides.append(Side(args.lender, args.borrower, cfg))
    for cap in [int(x) for x in args.ctas.split(",")]:
        for s in sides:
            s.ctx.set_option(aqua.OPT_PEER_CTAS, cap)
            s.enqueue(args.warmup, None)
        for s in sides:
            torch.cuda.synchronize(s.bdev)
        evs = [s.events(args.steps) for s in sides]
        for s, e in zip(sides, evs):
            s.enqueue(args.steps, e)
        for s in sides:
            torch.cuda.synchronize(s.bdev)
        recs = []
        for s, e in zip(sides, evs):
            out_ms = sorted(a.elapsed_time(b) for a, b, _ in e)
            in_ms = sorted(b.elapsed_time(c) for _, b, c in e)
            o, i = out_ms[len(out_ms) // 2], in_ms[len(in_ms) // 2]
            launch = s.ctx.last_launch()
            go, gi = s.nblk * s.U / (o / 1e3) / 1e9, s.nblk * s.U / (i / 1e3) / 1e9
            recs.append({"borrower": s.bdev, "lender": s.ldev, "probe": s.info["probe"],
                         "swap_out_GBps": round(go, 1), "swap_in_GBps": round(gi, 1),
                         "frac_of_900": [round(go / 900, 4), round(gi / 900, 4)],
                         "frac_of_770": [round(go / 770, 4), round(gi / 770, 4)],
                         "preempt_ms_p50": round(o, 4), "resume_ms_p50": round(i, 4),
                         "ctas": launch["ctas"], "engine": launch["engine"], "stages": launch["stages"],
                         "schedule": launch["schedule"], "verify_mismatches": s.verify()})
        print(json.dumps({"config": args.config, "peer_ctas": cap, "bidir": args.bidir,
                          "smoke_same_gpu": args.borrower == args.lender,
                          "bytes_per_direction": sides[0].nblk * sides[0].U, "pairs": recs}), flush=True)
    for s in sides:
        s.ctx.close()


if __name__ == "__main__":
    main()
