"""Tensor-parallel paging (BASELINE configs[3]): every TP rank
holds one KV-head shard of every prompt and pages its own shard.  The swap
lists must be identical across ranks; here each rank runs the same
deterministic native scheduler (no broadcast needed) on the bursty trace and
the ranks check that their call logs hash to the same value.

    torchrun --nproc-per-node 4 scripts/c3_tp.py            # one rank per GPU
    AQUA_BENCH_SHARED_GPU=1 torchrun --nproc-per-node 2 ...  # functional check on one GPU

Shape: Llama-3-70B KV (80 layers, 8 KV heads, D=128, bf16, block 16) split over
the TP ranks (8 / tp heads each); the lender is the same GPU (self) so the
run works on any box; the schedule is what is being checked.
"""
import hashlib
import json
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2407_21255_b200 import aqua  # noqa: E402
from paper_2407_21255_b200.cfs import Scheduler  # noqa: E402
from paper_2407_21255_b200.driver import run_trace  # noqa: E402
from workloads import burst_trace  # noqa: E402


def main():
    ws, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    shared = os.environ.get("AQUA_BENCH_SHARED_GPU") == "1"
    local = 0 if shared else int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    L, bs, D, H_total = 80, 16, 128, 8
    H = H_total // ws
    NB = 2048
    S = bs * H * D * 2
    U = 2 * L * S
    layers = [torch.zeros(2 * NB * S, dtype=torch.uint8, device="cuda") for _ in range(L)]
    ctx = aqua.Ctx(local, L, bs, H, D, 2, NB, [t.data_ptr() for t in layers])
    lend = 8 * NB * U
    arena = torch.empty(lend, dtype=torch.uint8, device="cuda")
    ctx.lend(local, arena.data_ptr(), lend)
    sched = Scheduler(NB=NB, bs=bs, b=512, k=8)
    trace = burst_trace(seed=1, burst_s=20.0, tail_s=5.0)
    t0 = time.perf_counter()
    log, st = run_trace(trace, ctx, sched, fill_seed=3)
    torch.cuda.synchronize()
    h = hashlib.sha256(repr(log).encode()).hexdigest()
    hashes = [None] * ws
    dist.all_gather_object(hashes, (rank, h, st["blocks_out"], st["iters"]))
    if rank == 0:
        same = len({x[1] for x in hashes}) == 1
        print(json.dumps({"tp": ws, "heads_per_rank": H, "U_bytes": U, "iterations": st["iters"],
                          "blocks_out_per_rank": st["blocks_out"], "identical_schedules": same,
                          "log_sha256": h, "wall_s": round(time.perf_counter() - t0, 2)}), flush=True)
        if not same:
            raise SystemExit("TP ranks diverged")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
