"""NEXT-4 over NVLink ("impact of sharing memory on producers";
P:1046-1049 "distributed producers" with TP all-reduce on the same links):

    python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \\
        --master-addr 127.0.0.1 --master-port 29511 scripts/nvlink_interference.py \\
        [--weights-gb 16] [--ctas 0,32,16,8] [--allreduce-mb 256]

Rank 1 is the lender (producer): it offers HBM through a CUDA IPC handle and
runs an HBM-bound decode proxy (one pass over W GB of "weights" per step,
16 GB ~ a Llama-3-8B bf16 decode step).  Rank 0 is the borrower (consumer):
it pages the C2 prompt (2 x 4 GiB) into the lender's HBM at link speed,
preempt + resume back to back.  For each borrower peer-CTA cap (the paging
budget, AQUA_OPT_PEER_CTAS) three phases, each started by a barrier:

  A  lender decode alone                      -> decode_alone_ms
  B  decode while the borrower pages into it  -> decode_with_paging_ms, paging GB/s per direction
  C  B + an NCCL all-reduce of --allreduce-mb looping on both ranks on a side
     stream (the TP collective sharing the same NVLink)   -> slowdowns, all-reduce bus GB/s

Rank 0 prints one JSON line per cap: the lender's decode slowdown against
the paging rate it bought, and the paging rate left under a
concurrent collective.  AQUA_BENCH_SHARED_GPU=1 runs both ranks on cuda:0
(gloo; no all-reduce phase) as a smoke test of the harness itself -- its
numbers are not NVLink numbers.
"""
import argparse
import json
import os
import statistics
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2407_21255_b200 import aqua  # noqa: E402
from paper_2407_21255_b200.pairing import exchange  # noqa: E402
from workloads import block_permutation  # noqa: E402

L, bs, H, D, NB, NBLK = 32, 16, 8, 128, 4096, 2048
S = bs * H * D * 2
U = 2 * L * S


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--weights-gb", type=float, default=16.0)
    ap.add_argument("--ctas", default="0,32,16,8")
    ap.add_argument("--allreduce-mb", type=int, default=256)
    ap.add_argument("--steps", type=int, default=6, help="decode steps per phase")
    args = ap.parse_args()
    shared = os.environ.get("AQUA_BENCH_SHARED_GPU") == "1"
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    assert ws == 2, "one borrower (rank 0) + one lender (rank 1)"
    local = 0 if shared else int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("gloo" if shared else "nccl", device_id=None if shared else dev)

    if rank == 1:
        ptr = aqua.ipc_alloc(local, NBLK * U)
        exchange(aqua.ipc_export(ptr))
        w = torch.ones(int(args.weights_gb * 1e9) // 8, dtype=torch.int64, device=dev)
        out = torch.empty((), dtype=torch.int64, device=dev)
        dec = torch.cuda.Stream(device=dev)
    else:
        handle = exchange(None)[1]
        layers = [torch.empty(2 * NB * S, dtype=torch.uint8, device=dev) for _ in range(L)]
        ctx = aqua.Ctx(local, L, bs, H, D, 2, NB, [t.data_ptr() for t in layers])
        mapped = aqua.ipc_import(local, handle)
        ctx.lend(aqua.MAPPED, mapped, NBLK * U)
        info = ctx.arena_info(aqua.LOC_PEER)
        perm = block_permutation(NB, NB, seed=2).tolist()
        ctx.adopt_blocks(1, perm[NBLK:])
        ctx.adopt_blocks(7, perm[:NBLK])
        ctx.kv_fill_pattern(7, 0, NBLK * bs, 99)
        swp = torch.cuda.Stream(device=dev)
    ar_buf = torch.ones(args.allreduce_mb << 18, dtype=torch.float32, device=dev)
    side = torch.cuda.Stream(device=dev)

    def decode_steps():
        evs = []
        for _ in range(args.steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(dec)
            with torch.cuda.stream(dec):
                torch.sum(w, dim=0, out=out)
            b.record(dec)
            evs.append((a, b))
        dec.synchronize()
        return statistics.median(a.elapsed_time(b) for a, b in evs)

    def page_until(flag_time):
        """Borrower: preempt + resume back to back until the wall clock passes flag_time."""
        outs, ins = [], []
        while time.time() < flag_time:
            a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a.record(swp)
            ctx.swap_out([7], swp.cuda_stream)
            b.record(swp)
            ctx.swap_in([7], swp.cuda_stream)
            c.record(swp)
            c.synchronize()
            outs.append(a.elapsed_time(b))
            ins.append(b.elapsed_time(c))
        return outs, ins

    def allreduce_loop(n):
        """n all-reduces back to back on the side stream (the same count on both ranks)."""
        t0 = time.time()
        with torch.cuda.stream(side):
            for _ in range(n):
                dist.all_reduce(ar_buf)
        side.synchronize()
        dt = time.time() - t0
        # bus bandwidth of a 2-rank all-reduce: 2 (n-1)/n x bytes / time = bytes / time
        return dt, (n * ar_buf.numel() * 4 / dt / 1e9) if dt > 0 else 0.0

    phase_s = 1.5
    n_ar = 0
    if not shared:                      # size the all-reduce loop to span a phase (same count on both ranks)
        allreduce_loop(3)
        dt, bus_alone = allreduce_loop(10)
        n_ar = max(10, int(phase_s / max(max(exchange(dt)) / 10, 1e-6)))
    for cap in [int(x) for x in args.ctas.split(",")]:
        res = {"peer_ctas": cap or "all"}
        # A: decode alone
        dist.barrier()
        if rank == 1:
            decode_steps()
            res["decode_alone_ms"] = decode_steps()
        if rank == 0 and not shared:
            res["allreduce_alone_busGBps"] = round(bus_alone, 1)
        # B: decode while the borrower pages into the lender; C: plus the all-reduce loop
        for phase, with_ar in (("B", False), ("C", True)):
            if with_ar and shared:
                continue
            dist.barrier()
            stop = exchange(time.time() + phase_s)[0]
            if with_ar:
                import threading
                ar_out = {}
                th = threading.Thread(target=lambda: ar_out.update(zip(("dt", "busbw"), allreduce_loop(n_ar))))
                th.start()
            if rank == 0:
                ctx.set_option(aqua.OPT_PEER_CTAS, cap)
                outs, ins = page_until(stop)
                res[f"{phase}_paging_GBps"] = [round(NBLK * U / (statistics.median(x) / 1e3) / 1e9, 1)
                                              for x in (outs, ins)]
            else:
                ms = []
                while time.time() < stop:
                    ms.append(decode_steps())
                res[f"{phase}_decode_ms"] = statistics.median(ms) if ms else None
            if with_ar:
                th.join()
                res[f"{phase}_allreduce_busGBps"] = round(ar_out.get("busbw", 0.0), 1)
        merged = {}
        for r in exchange(res):
            merged.update({k: v for k, v in r.items() if v is not None})
        if rank == 0:
            da = merged.get("decode_alone_ms")
            for phase in ("B", "C"):
                if da and merged.get(f"{phase}_decode_ms"):
                    merged[f"{phase}_decode_slowdown"] = round(merged[f"{phase}_decode_ms"] / da, 3)
            merged["lender_probe"] = info["probe"]
            merged["peer"] = info["peer"]
            merged["shared_gpu_smoke"] = shared
            print(json.dumps(merged), flush=True)
    dist.barrier()
    if rank == 0:
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        ctx.kv_verify_pattern(7, NBLK * bs, 99, cnt.data_ptr())
        torch.cuda.synchronize()
        ctx.close()
        aqua.ipc_close(local, mapped)
        print(json.dumps({"verify_mismatches": int(cnt.item())}), flush=True)
    dist.barrier()
    if rank == 1:
        aqua.ipc_free(local, ptr)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
