"""Engine / launch-shape sweep and the C5 bandwidth sweep on one GPU
(self-lender: arena in the same HBM, or the pinned host arena).

    python scripts/sweep.py engines   -> per (engine, piece, max_ctas): swap_out / swap_in GB/s for C2
    python scripts/sweep.py c5        -> block size 8..128 x blocks per launch 1..1024 (BASELINE configs[4])

Prints one JSON object per line; the oracle's bwfit is NOT used here (fits
are done in tests/analysis with oracle.bwfit).
"""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2407_21255_b200 import aqua  # noqa: E402
from workloads import block_permutation  # noqa: E402

ENG = {"tma": aqua.KERNEL_TMA, "ldst": aqua.KERNEL_LDST, "gather_temp": aqua.BASE_GATHER_TEMP,
       "per_chunk": aqua.BASE_PER_CHUNK, "ce_host": aqua.KERNEL_CE_HOST}


def setup(L, bs, H, D, NB, nblk, host=False, block_major=False):
    S = bs * H * D * 2
    U = 2 * L * S
    layers = [torch.zeros(2 * NB * S, dtype=torch.uint8, device="cuda") for _ in range(L)]
    ctx = aqua.Ctx(0, L, bs, H, D, 2, NB, [t.data_ptr() for t in layers],
                   S if block_major else 0, 2 * S if block_major else 0)
    arena = None
    if host:
        ctx.lend(aqua.HOST, 0, nblk * U)
    else:
        arena = torch.empty(nblk * U, dtype=torch.uint8, device="cuda")
        ctx.lend(0, arena.data_ptr(), nblk * U)
    perm = block_permutation(NB, NB, seed=2).tolist()
    ctx.adopt_blocks(1, perm[nblk:])
    ctx.adopt_blocks(7, perm[:nblk])
    return ctx, layers, arena, U


def time_tickets(ctx, reps, stream, sleep_cycles=2_000_000):
    """Device time of each copy from the library's timing events.  A ticket's
    start event is recorded before the library prepares the launch, so on an
    idle GPU it would also count the host's descriptor work and the launch
    call (~10 us with the 32 KiB parameter block, more for 32K-block calls);
    a ~1 ms sleep kernel queued first keeps the stream busy until the swap
    kernel is enqueued (swap_in already queues behind swap_out)."""
    ctx.set_option(aqua.OPT_TIMING, 1)
    outs, ins = [], []
    for _ in range(reps + 2):
        if sleep_cycles:
            with torch.cuda.stream(stream):
                torch.cuda._sleep(sleep_cycles)
        t1 = ctx.swap_out([7], stream.cuda_stream)
        _, t2 = ctx.swap_in([7], stream.cuda_stream)
        torch.cuda.synchronize()
        outs.append(ctx.ticket_elapsed(t1))
        ins.append(ctx.ticket_elapsed(t2))
    ctx.set_option(aqua.OPT_TIMING, 0)
    return statistics.median(outs[2:]), statistics.median(ins[2:])


def time_swaps(ctx, reps, stream):
    outs, ins = [], []
    for _ in range(2):
        ctx.swap_out([7], stream.cuda_stream)
        ctx.swap_in([7], stream.cuda_stream)
    torch.cuda.synchronize()
    for _ in range(reps):
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record(stream)
        ctx.swap_out([7], stream.cuda_stream)
        b.record(stream)
        ctx.swap_in([7], stream.cuda_stream)
        c.record(stream)
        torch.cuda.synchronize()
        outs.append(a.elapsed_time(b))
        ins.append(b.elapsed_time(c))
    return statistics.median(outs), statistics.median(ins)


def engines():
    L, bs, H, D, NB, nblk = 32, 16, 8, 128, 4096, 2048
    ctx, layers, arena, U = setup(L, bs, H, D, NB, nblk)
    s = torch.cuda.Stream()
    nbytes = nblk * U
    grid = [("tma", p, c) for p in (4096, 8192, 16384, 32768) for c in (0, 148, 296, 444)]
    grid += [("ldst", 0, c) for c in (0, 148, 296, 592)]
    grid += [("gather_temp", 0, 0)]
    for eng, piece, ctas in grid:
        ctx.set_option(aqua.OPT_KERNEL, ENG[eng])
        ctx.set_option(aqua.OPT_TMA_PIECE, piece)
        ctx.set_option(aqua.OPT_MAX_CTAS, ctas)
        o, i = time_swaps(ctx, 10, s)
        print(json.dumps({"engine": eng, "piece": piece, "max_ctas": ctas, "out_ms": round(o, 4),
                          "in_ms": round(i, 4), "out_hbm_GBps": round(2 * nbytes / o / 1e6, 1),
                          "in_hbm_GBps": round(2 * nbytes / i / 1e6, 1)}), flush=True)


def host_ctas():
    """How many SMs the host (PCIe) path needs: SMs left for decode."""
    L, bs, H, D, NB, nblk = 32, 16, 8, 128, 1024, 512
    ctx, layers, arena, U = setup(L, bs, H, D, NB, nblk, host=True)
    s = torch.cuda.Stream()
    for eng in ("tma", "ldst"):
        for ctas in (1, 2, 4, 8, 16, 32, 74, 148):
            ctx.set_option(aqua.OPT_KERNEL, ENG[eng])
            ctx.set_option(aqua.OPT_MAX_CTAS, ctas)
            o, i = time_tickets(ctx, 3, s)
            print(json.dumps({"host_ctas": ctas, "engine": eng, "out_GBps": round(nblk * U / o / 1e6, 2),
                              "in_GBps": round(nblk * U / i / 1e6, 2)}), flush=True)


def host_pcie():
    """Host (PCIe) zero-copy path for an ncu capture: the TMA kernel writes
    and reads a 1 GiB image in pinned host memory (C2 shape, 512 blocks)."""
    L, bs, H, D, NB, nblk = 32, 16, 8, 128, 1024, 512
    ctx, layers, arena, U = setup(L, bs, H, D, NB, nblk, host=True)
    ctx.set_option(aqua.OPT_KERNEL, ENG["tma"])
    s = torch.cuda.Stream()
    o, i = time_tickets(ctx, 2, s)
    print(json.dumps({"host_pcie": nblk * U, "out_GBps": round(nblk * U / o / 1e6, 2),
                      "in_GBps": round(nblk * U / i / 1e6, 2)}), flush=True)


def self_ctas():
    """CTAs (SMs) needed to saturate HBM on the self-lender path."""
    L, bs, H, D, NB, nblk = 32, 16, 8, 128, 4096, 2048
    ctx, layers, arena, U = setup(L, bs, H, D, NB, nblk)
    s = torch.cuda.Stream()
    for ctas in (8, 16, 32, 48, 64, 96, 128, 148):
        ctx.set_option(aqua.OPT_MAX_CTAS, ctas)
        o, i = time_tickets(ctx, 5, s)
        print(json.dumps({"self_ctas": ctas, "out_hbm_GBps": round(2 * nblk * U / o / 1e6, 1),
                          "in_hbm_GBps": round(2 * nblk * U / i / 1e6, 1)}), flush=True)


def migrate():
    """NEXT-1 data path: a 4 GiB image moved lender -> host (reclaim) and
    host -> lender (re-offer), device time from the library's timing events."""
    L, bs, H, D, NB, nblk = 32, 16, 8, 128, 4096, 2048
    for engine in ("auto", "tma"):
        _migrate_one(engine, L, bs, H, D, NB, nblk)


def _migrate_one(engine, L, bs, H, D, NB, nblk):
    """AUTO moves the slot-contiguous images on the copy engines (no SMs);
    "tma" forces the fused arena->arena kernel (8 CTAs, the round-1 path)."""
    ctx, layers, arena, U = setup(L, bs, H, D, NB, nblk)
    ctx.lend(aqua.HOST, 0, nblk * U)
    if engine == "tma":
        ctx.set_option(aqua.OPT_KERNEL, aqua.KERNEL_TMA)
    ctx.set_option(aqua.OPT_TIMING, 1)
    s = torch.cuda.Stream()
    ctx.kv_fill_pattern(7, 0, nblk * bs, 5)
    ctx.swap_out([7], s.cuda_stream)
    res = []
    for rep in range(3):
        t1 = ctx.migrate([7], aqua.LOC_HOST, s.cuda_stream)
        t2 = ctx.migrate([7], aqua.LOC_PEER, s.cuda_stream)
        torch.cuda.synchronize()
        res.append((ctx.ticket_elapsed(t1), ctx.ticket_elapsed(t2)))
    t3 = ctx.reclaim(s.cuda_stream)
    torch.cuda.synchronize()
    rec = ctx.ticket_elapsed(t3)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    res_in = []
    for rep in range(3):   # resume from DRAM (the lender is gone), then page out there again
        _, t4 = ctx.swap_in([7], s.cuda_stream)
        ctx.kv_verify_pattern(7, nblk * bs, 5, cnt.data_ptr(), s.cuda_stream)
        torch.cuda.synchronize()
        res_in.append(ctx.ticket_elapsed(t4))
        if rep < 2:
            ctx.swap_out([7], s.cuda_stream)
    o = statistics.median(r[0] for r in res)
    i = statistics.median(r[1] for r in res)
    print(json.dumps({"engine": engine, "migrate_bytes": nblk * U, "to_host_ms": round(o, 3), "to_lender_ms": round(i, 3),
                      "to_host_GBps": round(nblk * U / o / 1e6, 2), "to_lender_GBps": round(nblk * U / i / 1e6, 2),
                      "reclaim_ms": round(rec, 3), "resume_from_host_ms": [round(x, 3) for x in res_in],
                      "verify_mismatches": int(cnt.item())}), flush=True)
    ctx.close()
    del layers, arena
    torch.cuda.empty_cache()


def prefix():
    """NEXT-2, BASELINE-adjacent E7 shape: Yi-34B-200K over TP2 per
    rank (60 layers, 4 KV heads, D=128, bf16, block 16 -> U = 1.875 MiB); a
    100K-token cached prefix (6250 blocks, 11.4 GiB) stored once and loaded on
    each hit, from the lender (self) and from host DRAM."""
    L, bs, H, D = 60, 16, 4, 128
    S = bs * H * D * 2
    U = 2 * L * S
    nblk = 6250
    NB = 2 * nblk + 64
    layers = [torch.zeros(2 * NB * S, dtype=torch.uint8, device="cuda") for _ in range(L)]
    out = {}
    for where in ("self", "host"):
        ctx = aqua.Ctx(0, L, bs, H, D, 2, NB, [t.data_ptr() for t in layers])
        arena = None
        if where == "self":
            arena = torch.empty(nblk * U, dtype=torch.uint8, device="cuda")
            ctx.lend(0, arena.data_ptr(), nblk * U)
        else:
            ctx.lend(aqua.HOST, 0, nblk * U)
        ctx.set_option(aqua.OPT_TIMING, 1)
        s = torch.cuda.Stream()
        ctx.adopt_blocks(1, block_permutation(NB, nblk, seed=4).tolist())
        ctx.kv_fill_pattern(1, 0, nblk * bs, 11, s.cuda_stream)
        t0 = ctx.prefix_store(77, 1, nblk, s.cuda_stream)
        torch.cuda.synchronize()
        store_ms = ctx.ticket_elapsed(t0)
        ctx.free(1, s.cuda_stream)
        loads = []
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        for hit in range(4):
            ids, tk = ctx.prefix_load(77, 1000 + hit, s.cuda_stream)
            torch.cuda.synchronize()
            loads.append(ctx.ticket_elapsed(tk))
            ctx.free(1000 + hit, s.cuda_stream)
        out[where] = {"store_ms": round(store_ms, 3), "load_ms_p50": round(statistics.median(loads), 3),
                      "load_GBps": round(nblk * U / statistics.median(loads) / 1e6, 1)}
        ctx.close()
        del arena
        torch.cuda.empty_cache()
    print(json.dumps({"prefix_tokens": nblk * bs, "bytes": nblk * U, **out}), flush=True)


def layers():
    """NEXT-3: layer-wise resume of an OPT-30B-like
    8192-token prompt (48 layers, 56 KV heads, D=128, bf16, block 16 -> U = 21
    MiB/block, 10.7 GiB: the paper's "10 GB swap space for an 8K prompt",
    P:1077) and of the C2 prompt; per-layer tickets give the time until layer 0
    is usable vs the whole resume, from the lender (self) and from host DRAM."""
    import time
    for name, (L, bs, H, D, nblk) in {"opt30b_8k": (48, 16, 56, 128, 512),
                                      "llama8b_32k": (32, 16, 8, 128, 2048)}.items():
        S = bs * H * D * 2
        U = 2 * L * S
        NB = 2 * nblk
        lay = [torch.zeros(2 * NB * S, dtype=torch.uint8, device="cuda") for _ in range(L)]
        for where in ("self", "host"):
            ctx = aqua.Ctx(0, L, bs, H, D, 2, NB, [t.data_ptr() for t in lay])
            arena = None
            if where == "self":
                arena = torch.empty(nblk * U, dtype=torch.uint8, device="cuda")
                ctx.lend(0, arena.data_ptr(), nblk * U)
            else:
                ctx.lend(aqua.HOST, 0, nblk * U)
            ctx.set_option(aqua.OPT_TIMING, 1)
            s = torch.cuda.Stream()
            perm = block_permutation(NB, NB, seed=2).tolist()
            ctx.adopt_blocks(1, perm[nblk:])
            ctx.adopt_blocks(7, perm[:nblk])
            rows = []
            for rep in range(3):
                ctx.swap_out([7], s.cuda_stream)
                torch.cuda.synchronize()
                a = torch.cuda.Event(enable_timing=True)
                a.record(s)
                new, tks = ctx.swap_in_layers([7], 1, s.cuda_stream)
                torch.cuda.synchronize()
                per = [ctx.ticket_elapsed(t) for t in tks]
                rows.append((per[0], sum(per)))
            first = statistics.median(r[0] for r in rows)
            total = statistics.median(r[1] for r in rows)
            print(json.dumps({"layers": name, "where": where, "bytes": nblk * U, "L": L,
                              "first_layer_ms": round(first, 3), "all_layers_ms": round(total, 3),
                              "GBps": round(nblk * U / total / 1e6, 1)}), flush=True)
            ctx.close()
            del arena
            torch.cuda.empty_cache()
        del lay
        torch.cuda.empty_cache()


def ctas_stages():
    """Per-SM efficiency when the swap is capped to few SMs (to leave the
    rest to decode): does a deeper ring recover throughput per SM?"""
    L, bs, H, D, NB, nblk = 32, 16, 8, 128, 4096, 2048
    ctx, layers, arena, U = setup(L, bs, H, D, NB, nblk)
    s = torch.cuda.Stream()
    for ctas in (8, 16, 32, 64):
        for st in (3, 4, 6):
            ctx.set_option(aqua.OPT_MAX_CTAS, ctas)
            ctx.set_option(aqua.OPT_TMA_STAGES, st)
            o, i = time_tickets(ctx, 3, s)
            print(json.dumps({"ctas": ctas, "stages": st, "out_hbm_GBps": round(2 * nblk * U / o / 1e6, 1),
                              "in_hbm_GBps": round(2 * nblk * U / i / 1e6, 1),
                              "per_sm_GBps": round(2 * nblk * U / o / 1e6 / ctas, 1)}), flush=True)


def c5_multi():
    """C5 at N >= 2 (torchrun): every rank pages into HBM lent by its partner
    over NVLink (IPC), all pairs at once; per point the device time of each
    call is the max over ranks.  AQUA_BENCH_SHARED_GPU=1 runs all ranks on
    cuda:0 (a functional check of the multi-rank path on one GPU)."""
    import torch.distributed as dist
    from paper_2407_21255_b200.pairing import best_matching, exchange
    ws, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    shared = os.environ.get("AQUA_BENCH_SHARED_GPU") == "1"
    local = 0 if shared else int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    row = [0.0 if j == local else (1.0 if shared or aqua.can_access_peer(local, j) else 0.0) for j in range(ws)]
    partner = best_matching(exchange(row))[rank]
    L, H, D = 32, 8, 128
    for bs in (8, 16, 32, 64, 128):
        S = bs * H * D * 2
        U = 2 * L * S
        for nblk in (1, 4, 16, 64, 256, 1024):
            if nblk * U > (8 << 30):
                continue
            mine = aqua.ipc_alloc(local, nblk * U)
            got = exchange((aqua.ipc_export(mine), nblk * U))
            NB = 2 * nblk
            layers = [torch.zeros(2 * NB * S, dtype=torch.uint8, device="cuda") for _ in range(L)]
            ctx = aqua.Ctx(local, L, bs, H, D, 2, NB, [t.data_ptr() for t in layers])
            mapped = None
            if partner == rank:
                ctx.lend(local, mine, nblk * U)
            else:
                mapped = aqua.ipc_import(local, got[partner][0])
                ctx.lend(aqua.MAPPED, mapped, nblk * U)
            perm = block_permutation(NB, NB, seed=2).tolist()
            ctx.adopt_blocks(1, perm[nblk:])
            ctx.adopt_blocks(7, perm[:nblk])
            s = torch.cuda.Stream()
            dist.barrier()
            o, i = time_tickets(ctx, 5, s)
            t = torch.tensor([o, i], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            if rank == 0:
                print(json.dumps({"c5_multi": ws, "partner0": partner, "bs": bs, "blocks": nblk, "bytes": nblk * U,
                                  "out_ms_max": round(float(t[0]), 5), "in_ms_max": round(float(t[1]), 5),
                                  "out_GBps": round(nblk * U / float(t[0]) / 1e6, 2),
                                  "in_GBps": round(nblk * U / float(t[1]) / 1e6, 2)}), flush=True)
            ctx.close()
            if mapped:
                aqua.ipc_close(local, mapped)
            dist.barrier()
            aqua.ipc_free(local, mine)
            del layers
            torch.cuda.empty_cache()
    dist.destroy_process_group()


def torch_baseline():
    """What a PyTorch user would write for the same swap: per layer, index the
    [2][NB][S] pool view with the block table and copy into the slot-major
    arena view (L*2 gather/scatter ops), vs the fused kernel."""
    L, bs, H, D, NB, nblk = 32, 16, 8, 128, 4096, 2048
    ctx, layers, arena, U = setup(L, bs, H, D, NB, nblk)
    S = bs * H * D * 2
    bt = torch.tensor(block_permutation(NB, NB, seed=2)[:nblk].tolist(), device="cuda", dtype=torch.int64)
    img = arena.view(nblk, L, 2, S)
    views = [t.view(2, NB, S) for t in layers]

    def out():
        for l in range(L):
            img[:, l] = views[l][:, bt].transpose(0, 1)

    def inn():
        for l in range(L):
            views[l][:, bt] = img[:, l].transpose(0, 1)

    res = {}
    for name, fn in (("torch_swap_out", out), ("torch_swap_in", inn)):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res[name] = {"ms": round(statistics.median(ts), 3),
                     "hbm_GBps": round(2 * nblk * U / statistics.median(ts) / 1e6, 1)}
    o, i = time_tickets(ctx, 5, torch.cuda.Stream())
    res["aqua_tma"] = {"out_ms": round(o, 3), "in_ms": round(i, 3)}
    print(json.dumps(res), flush=True)


def exchange():
    """Preempt prompt A + resume prompt B (2048 blocks each, C2 shape) as two
    sequential calls vs one aqua_swap_exchange on two streams, for the
    lender-in-HBM and the host-DRAM arenas (full-duplex PCIe)."""
    import time
    L, bs, H, D, NB = 32, 16, 8, 128, 6144
    nblk = 2048
    S = bs * H * D * 2
    U = 2 * L * S
    layers = [torch.zeros(2 * NB * S, dtype=torch.uint8, device="cuda") for _ in range(L)]
    for where in ("self", "host"):
        ctx = aqua.Ctx(0, L, bs, H, D, 2, NB, [t.data_ptr() for t in layers])
        arena = None
        if where == "self":
            arena = torch.empty(2 * nblk * U, dtype=torch.uint8, device="cuda")
            ctx.lend(0, arena.data_ptr(), 2 * nblk * U)
        else:
            ctx.lend(aqua.HOST, 0, 2 * nblk * U)
        perm = block_permutation(NB, NB, seed=2).tolist()
        ctx.adopt_blocks(1, perm[2 * nblk:])
        ctx.adopt_blocks(7, perm[:nblk])
        ctx.adopt_blocks(8, perm[nblk:2 * nblk])
        ctx.swap_out([8])
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        res = {}
        for mode in ("sequential", "exchange"):
            ts = []
            for rep in range(4):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                if mode == "sequential":
                    ctx.swap_out([7], s1.cuda_stream)
                    ctx.swap_in([8], s1.cuda_stream)
                    ctx.swap_out([8], s1.cuda_stream)
                    ctx.swap_in([7], s1.cuda_stream)
                else:
                    ctx.swap_exchange([7], [8], s1.cuda_stream, s2.cuda_stream, pieces=8)
                    ctx.swap_exchange([8], [7], s2.cuda_stream, s1.cuda_stream, pieces=8)
                torch.cuda.synchronize()
                ts.append((time.perf_counter() - t0) / 2)
            res[mode] = round(1e3 * statistics.median(ts[1:]), 3)
        print(json.dumps({"exchange": where, "bytes_each_way": nblk * U, "ms_per_reschedule": res,
                          "speedup": round(res["sequential"] / res["exchange"], 3)}), flush=True)
        ctx.close()
        del arena
        torch.cuda.empty_cache()


def duplex():
    """Is the host link full duplex?  Copy-engine H2D + D2H concurrently vs
    alone (1 GiB pinned each), and the zero-copy exchange at several piece
    counts and CTA caps."""
    n = 1 << 30
    h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def run(both):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        s1.wait_event(a)
        s2.wait_event(a)
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
        if both:
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
        e1, e2 = torch.cuda.Event(), torch.cuda.Event()
        e1.record(s1)
        e2.record(s2)
        torch.cuda.current_stream().wait_event(e1)
        torch.cuda.current_stream().wait_event(e2)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b)
    run(True)
    alone = min(run(False) for _ in range(3))
    both = min(run(True) for _ in range(3))
    print(json.dumps({"duplex_ce": {"h2d_alone_GBps": round(n / alone / 1e6, 1),
                                    "h2d_plus_d2h_total_GBps": round(2 * n / both / 1e6, 1)}}), flush=True)
    L, bs, H, D, NB = 32, 16, 8, 128, 6144
    nblk = 2048
    S = bs * H * D * 2
    U = 2 * L * S
    layers = [torch.zeros(2 * NB * S, dtype=torch.uint8, device="cuda") for _ in range(L)]
    ctx = aqua.Ctx(0, L, bs, H, D, 2, NB, [t.data_ptr() for t in layers])
    ctx.lend(aqua.HOST, 0, 2 * nblk * U)
    perm = block_permutation(NB, NB, seed=2).tolist()
    ctx.adopt_blocks(1, perm[2 * nblk:])
    ctx.adopt_blocks(7, perm[:nblk])
    ctx.adopt_blocks(8, perm[nblk:2 * nblk])
    ctx.swap_out([8])
    import time
    for eng, ctas in (("tma", 8), ("tma", 16), ("ce_host", 0)):
        ctx.set_option(aqua.OPT_KERNEL, ENG[eng] if eng in ENG else aqua.KERNEL_CE_HOST)
        ctx.set_option(aqua.OPT_MAX_CTAS, ctas)
        for pieces in (1, 4, 16):
            ts = []
            for rep in range(3):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                ctx.swap_exchange([7], [8], s1.cuda_stream, s2.cuda_stream, pieces=pieces)
                ctx.swap_exchange([8], [7], s2.cuda_stream, s1.cuda_stream, pieces=pieces)
                torch.cuda.synchronize()
                ts.append((time.perf_counter() - t0) / 2)
            ms = 1e3 * statistics.median(ts)
            print(json.dumps({"host_exchange_engine": eng, "ctas": ctas, "pieces": pieces, "ms": round(ms, 2),
                              "total_GBps": round(2 * nblk * U / ms / 1e6, 1)}), flush=True)


def layer_overlap():
    """NEXT-3 in use: a decode that walks the layers of a resumed prompt.
    (a) wait for the whole resume, then run 32 per-layer decode steps;
    (b) resume with per-layer tickets and start layer l as soon as ticket l
    completes.  Decode proxy per layer: a reduction over `per_layer_mb` of
    HBM (a layer's weights).  Lender in HBM and host DRAM."""
    L, bs, H, D, NB, nblk = 32, 16, 8, 128, 4096, 2048
    per_layer_mb = 512
    w = torch.ones(L * per_layer_mb * (1 << 20) // 8, dtype=torch.int64, device="cuda").view(L, -1)
    out = torch.empty((), dtype=torch.int64, device="cuda")
    for where in ("self", "host"):
        ctx, layers, arena, U = setup(L, bs, H, D, NB, nblk, host=(where == "host"))
        dec, swp = torch.cuda.Stream(), torch.cuda.Stream()

        def decode_layer(l):
            with torch.cuda.stream(dec):
                torch.sum(w[l], dim=0, out=out)

        res = {}
        for mode in ("whole", "layerwise", "compute_only"):
            ts = []
            for rep in range(4):
                ctx.swap_out([7], swp.cuda_stream)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(dec)
                swp.wait_stream(dec)
                if mode == "whole":
                    _, tk = ctx.swap_in([7], swp.cuda_stream)
                    ctx.wait(tk, dec.cuda_stream)
                    for l in range(L):
                        decode_layer(l)
                elif mode == "layerwise":
                    _, tks = ctx.swap_in_layers([7], 1, swp.cuda_stream)
                    for l in range(L):
                        ctx.wait(tks[l], dec.cuda_stream)
                        decode_layer(l)
                else:
                    _, tk = ctx.swap_in([7], swp.cuda_stream)
                    for l in range(L):
                        decode_layer(l)
                b.record(dec)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            res[mode] = round(statistics.median(ts[1:]), 3)
        print(json.dumps({"layer_overlap": where, "per_layer_decode_MB": per_layer_mb, "ms": res}), flush=True)
        ctx.close()
        del arena, layers
        torch.cuda.empty_cache()


def tma_variants():
    """TMA engine: the ring (0) vs the hybrid ring + LDST warps (3), C2
    self-lender, across ring depths and SM caps; LDST for reference."""
    L, bs, H, D, NB, nblk = 32, 16, 8, 128, 4096, 2048
    ctx, layers, arena, U = setup(L, bs, H, D, NB, nblk)
    s = torch.cuda.Stream()
    vs = [int(x) for x in os.environ.get("AQUA_SWEEP_TMA_VARIANTS", "0,3").split(",")]
    sts = [int(x) for x in os.environ.get("AQUA_SWEEP_STAGES", "0,2,3,4,6").split(",")]
    for v in vs:
        for st in sts:
            for ctas in (0, 74, 32, 16):
                ctx.set_option(aqua.OPT_KERNEL, aqua.KERNEL_TMA)
                ctx.set_option(aqua.OPT_TMA_VARIANT, v)
                ctx.set_option(aqua.OPT_TMA_STAGES, st)
                ctx.set_option(aqua.OPT_MAX_CTAS, ctas)
                o, i = time_tickets(ctx, 5, s)
                print(json.dumps({"tma_variant": v, "stages": st or "auto", "ctas": ctas or 148,
                                  "out_hbm_GBps": round(2 * nblk * U / o / 1e6, 1),
                                  "in_hbm_GBps": round(2 * nblk * U / i / 1e6, 1)}), flush=True)
    ctx.set_option(aqua.OPT_TMA_STAGES, 0)
    ctx.set_option(aqua.OPT_KERNEL, aqua.KERNEL_LDST)
    for ctas in (0, 74, 32, 16):
        ctx.set_option(aqua.OPT_MAX_CTAS, ctas)
        o, i = time_tickets(ctx, 5, s)
        print(json.dumps({"ldst_variant": 2, "ctas": ctas or 148, "out_hbm_GBps": round(2 * nblk * U / o / 1e6, 1),
                          "in_hbm_GBps": round(2 * nblk * U / i / 1e6, 1)}), flush=True)


def time_queued(ctx, stream, K=10, reps=3):
    """Back-to-back device time per swap_out + swap_in pair, the calls queued
    behind a sleep kernel (no host gaps): min over reps of (end - start) / K."""
    best = 1e30
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            torch.cuda._sleep(20_000_000)
        a.record(stream)
        for _ in range(K):
            ctx.swap_out([7], stream.cuda_stream)
            ctx.swap_in([7], stream.cuda_stream)
        b.record(stream)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / K)
    return best


def tma_sched():
    """TMA engine work distribution: static contiguous ranges (0), claimed
    batches of n ring units (n > 0); C2 and the C4 (70B/TP4, S = 8 KiB)
    shape, all SMs and SM caps; back-to-back (queued) and per-call (ticket)
    device times.  AQUA_SWEEP_SCHED = "n,...", AQUA_SWEEP_CTAS = "0,64,16"."""
    combos = [(int(x), 0) for x in os.environ.get("AQUA_SWEEP_SCHED", "0,1,2,4,8,16").split(",")]
    ctas_list = [int(x) for x in os.environ.get("AQUA_SWEEP_CTAS", "0,64,16").split(",")]
    stages_list = [int(x) for x in os.environ.get("AQUA_SWEEP_STAGES", "0").split(",")]
    pieces = [int(x) for x in os.environ.get("AQUA_SWEEP_PIECES", "0").split(",")]
    for name, (L, H, nblk) in (("c2", (32, 8, 2048)), ("c4", (80, 2, 4096))):
        ctx, layers, arena, U = setup(L, 16, H, 128, 2 * nblk, nblk)
        s = torch.cuda.Stream()
        ctx.set_option(aqua.OPT_KERNEL, aqua.KERNEL_TMA)
        for ctas in ctas_list:
            ctx.set_option(aqua.OPT_MAX_CTAS, ctas)
            for sc, pct in combos:
              for st in stages_list:
               for pc in pieces:
                ctx.set_option(aqua.OPT_TMA_PIECE, pc)
                ctx.set_option(aqua.OPT_TMA_SCHED, sc)
                ctx.set_option(aqua.OPT_TMA_STAGES, st)
                pair = time_queued(ctx, s, K=20, reps=5)
                o, i = time_tickets(ctx, 5, s)
                print(json.dumps({"tma_sched": sc, "static_pct": pct, "stages": st or "auto", "piece": pc or 32768,
                                  "shape": name,
                                  "ctas": ctas or 148,
                                  "pair_ms": round(pair, 4), "swap_GBps": round(2 * nblk * U / pair / 1e6, 1),
                                  "hbm_GBps": round(4 * nblk * U / pair / 1e6, 1),
                                  "out_hbm_GBps": round(2 * nblk * U / o / 1e6, 1),
                                  "in_hbm_GBps": round(2 * nblk * U / i / 1e6, 1)}), flush=True)
        ctx.close()
        del layers, arena
        torch.cuda.empty_cache()


def hybrid():
    """TMA ring alone (variant 0) vs ring + 8 LDST warps (variant 3) under SM
    caps, C2 and C4 shapes, back-to-back device time."""
    for name, (L, H, nblk) in (("c2", (32, 8, 2048)), ("c4", (80, 2, 4096))):
        ctx, layers, arena, U = setup(L, 16, H, 128, 2 * nblk, nblk)
        s = torch.cuda.Stream()
        ctx.set_option(aqua.OPT_KERNEL, aqua.KERNEL_TMA)
        for ctas in (148, 96, 64, 32, 16, 8):
            ctx.set_option(aqua.OPT_MAX_CTAS, ctas)
            for v, sc in ((0, aqua.TMA_SCHED_AUTO), (0, 2), (3, 2), (3, 8)):
                ctx.set_option(aqua.OPT_TMA_VARIANT, v)
                ctx.set_option(aqua.OPT_TMA_SCHED, sc)
                pair = time_queued(ctx, s, K=10, reps=3)
                print(json.dumps({"hybrid": v, "sched": "auto" if sc == aqua.TMA_SCHED_AUTO else sc, "shape": name,
                                  "ctas": ctas, "pair_ms": round(pair, 4),
                                  "hbm_GBps": round(4 * nblk * U / pair / 1e6, 1),
                                  "per_sm_GBps": round(4 * nblk * U / pair / 1e6 / ctas, 1)}), flush=True)
        ctx.close()
        del layers, arena
        torch.cuda.empty_cache()


def small_chunks():
    """Sub-stage chunks at full grid and under a cap: S = 512 B .. 8 KiB (e.g. one
    KV head per TP8 rank: S = 4 KiB), TMA ring vs hybrid, 1 GiB per call.
    AQUA_SWEEP_BLOCK_MAJOR=1: the block-major layout (K and V of a layer
    adjacent: moved as one 2S chunk)."""
    bm = os.environ.get("AQUA_SWEEP_BLOCK_MAJOR") == "1"
    for H, D in ((1, 16), (1, 32), (1, 64), (1, 128), (2, 128)):
        L = 32
        S = 16 * H * D * 2
        U = 2 * L * S
        nblk = (1 << 30) // U
        ctx, layers, arena, _ = setup(L, 16, H, D, 2 * nblk, nblk, block_major=bm)
        s = torch.cuda.Stream()
        ctx.set_option(aqua.OPT_KERNEL, aqua.KERNEL_TMA)
        for ctas in (148, 32):
            ctx.set_option(aqua.OPT_MAX_CTAS, ctas)
            for v, sc in ((0, aqua.TMA_SCHED_AUTO), (0, 2), (0, 8), (3, 2), (3, 8), (3, 16)):
                ctx.set_option(aqua.OPT_TMA_VARIANT, v)
                ctx.set_option(aqua.OPT_TMA_SCHED, sc)
                pair = time_queued(ctx, s, K=10, reps=3)
                print(json.dumps({"S": S, "block_major": bm, "variant": v,
                                  "sched": "auto" if sc == aqua.TMA_SCHED_AUTO else sc,
                                  "ctas": ctas, "launch": ctx.last_launch()["schedule"],
                                  "hbm_GBps": round(4 * nblk * U / pair / 1e6, 1)}), flush=True)
        ctx.set_option(aqua.OPT_TMA_VARIANT, 0)
        ctx.close()
        del layers, arena
        torch.cuda.empty_cache()


def small_chunks2():
    """Round 2: sub-stage chunks (plane-major, S = 512 B .. 8 KiB, 1 GiB per
    call): the TMA ring with claimed batches of n units (the warp's lanes
    issue a unit's pool-side copies) and the hybrid ring + LDST warps; all
    SMs and a 32-SM cap.  (The register movers alone and a staged kernel --
    TMA for the image side only, registers for the pool side -- were
    measured with this sweep and removed: profiles/r02_small_chunks_*.jsonl.)"""
    Ss = [int(x) for x in os.environ.get("AQUA_SWEEP_S", "512,1024,2048,4096,8192").split(",")]
    for S in Ss:
        L, H = 32, 1
        D = S // 32 if S <= 4096 else 128
        if S > 4096:
            H = S // 4096
        U = 2 * L * S
        nblk = (1 << 30) // U
        bm = os.environ.get("AQUA_SWEEP_BLOCK_MAJOR") == "1"
        ctx, layers, arena, _ = setup(L, 16, H, D, 2 * nblk, nblk, block_major=bm)
        s = torch.cuda.Stream()
        for cap in (0, 32):
            combos = [("ring", 0, 0, n) for n in (2, 4, 8, 16, 32)]
            combos += [("hybrid", 0, 3, n) for n in (1, 2, 4)]
            combos += [("auto", 0, 0, aqua.TMA_SCHED_AUTO)]
            only = os.environ.get("AQUA_SWEEP_ENGINES")
            if only:
                combos = [x for x in combos if x[0] in only.split(",")]
            hyb_n = os.environ.get("AQUA_SWEEP_HYBRID_UNITS")
            if hyb_n:
                combos = [x for x in combos if x[0] != "hybrid"] + [("hybrid", 0, 3, int(n)) for n in hyb_n.split(",")]
            st_list = [int(x) for x in os.environ.get("AQUA_SWEEP_RING_STAGES", "0").split(",")]
            combos = [(e, st, v, n) for (e, _, v, n) in combos for st in st_list]
            for eng, stg, v, n in combos:
                ctx.set_option(aqua.OPT_TMA_STAGES, stg)
                ctx.set_option(aqua.OPT_KERNEL, aqua.KERNEL_AUTO if eng == "auto" else aqua.KERNEL_TMA)
                ctx.set_option(aqua.OPT_TMA_VARIANT, v)
                ctx.set_option(aqua.OPT_TMA_SCHED, n)
                ctx.set_option(aqua.OPT_MAX_CTAS, cap)
                pair = time_queued(ctx, s, K=10, reps=3)
                ll = ctx.last_launch()
                print(json.dumps({"S": S, "block_major": bm, "cap": cap or 148, "engine": eng, "sched_units": n,
                                  "grid": ll["ctas"],
                                  "kernel": ll["engine"], "variant": ll["variant"],
                                  "ldst_units": int(os.environ.get("AQUA_HYBRID_LDST_UNITS", "0")),
                                  "stages": ll["stages"],
                                  "threads": ll["threads_per_cta"], "launch": ll["schedule"],
                                  "hbm_GBps": round(4 * nblk * U / pair / 1e6, 1)}), flush=True)
        ctx.set_option(aqua.OPT_TMA_VARIANT, 0)
        ctx.set_option(aqua.OPT_TMA_SCHED, aqua.TMA_SCHED_AUTO)
        ctx.set_option(aqua.OPT_TMA_STAGES, 0)
        ctx.close()
        del layers, arena
        torch.cuda.empty_cache()


def small_ldst_sweep():
    """The small-chunk register kernel (LDST variant 3) vs AUTO, the ring and
    the hybrid, S = 512 B .. 4 KiB, 1 GiB calls, all SMs and a 32-CTA cap.
    Two clocks: `queued` = back-to-back calls from Python (host bookkeeping and
    the binding's id lists included: with 512 B chunks a 1 GiB call is 32,768
    blocks and the host side takes longer than the kernel), `device` = each
    call's device time from the library's timing events (descriptor upload +
    kernel)."""
    Ss = [int(x) for x in os.environ.get("AQUA_SWEEP_S", "512,1024,2048,4096").split(",")]
    for S in Ss:
        L, H, D = 32, 1, S // 32
        U = 2 * L * S
        nblk = (1 << 30) // U
        ctx, layers, arena, _ = setup(L, 16, H, D, 2 * nblk, nblk)
        s = torch.cuda.Stream()
        for eng, cap in (("auto", 0), ("small", 0), ("ring", 0), ("hybrid", 0), ("auto", 32), ("small", 32)):
            ctx.set_option(aqua.OPT_KERNEL, {"auto": aqua.KERNEL_AUTO, "small": aqua.KERNEL_LDST}.get(eng, aqua.KERNEL_TMA))
            ctx.set_option(aqua.OPT_LDST_VARIANT, 3 if eng == "small" else 2)
            ctx.set_option(aqua.OPT_TMA_VARIANT, 3 if eng == "hybrid" else 0)
            ctx.set_option(aqua.OPT_MAX_CTAS, cap)
            pair = time_queued(ctx, s, K=10, reps=3)
            o, i = time_tickets(ctx, 5, s)
            ll = ctx.last_launch()
            print(json.dumps({"S": S, "engine": eng, "cap": cap, "kernel": ll["engine"], "grid": ll["ctas"],
                              "variant": ll["variant"], "launch": ll["schedule"],
                              "hbm_GBps_queued": round(4 * nblk * U / pair / 1e6, 1),
                              "hbm_GBps_device_out": round(2 * nblk * U / o / 1e6, 1),
                              "hbm_GBps_device_in": round(2 * nblk * U / i / 1e6, 1)}), flush=True)
        ctx.set_option(aqua.OPT_TMA_VARIANT, 0)
        ctx.close()
        del layers, arena
        torch.cuda.empty_cache()


def rate():
    """AQUA_OPT_RATE_GBPS: achieved swap GB/s per direction against the budget
    (C2 and C4 shapes, back to back)."""
    for name, (L, H, nblk) in (("c2", (32, 8, 2048)), ("c4", (80, 2, 4096))):
        ctx, layers, arena, U = setup(L, 16, H, 128, 2 * nblk, nblk)
        s = torch.cuda.Stream()
        for r in (100, 200, 400, 800, 1600, 3200, 0):
            ctx.set_option(aqua.OPT_RATE_GBPS, r)
            pair = time_queued(ctx, s, K=6, reps=3)
            ctx.swap_out([7], s.cuda_stream)
            ctas = ctx.last_launch()["ctas"]
            ctx.swap_in([7], s.cuda_stream)
            torch.cuda.synchronize()
            print(json.dumps({"rate_budget_GBps": r or None, "shape": name, "ctas": ctas,
                              "swap_GBps_per_direction": round(2 * nblk * U / pair / 1e6, 1)}), flush=True)
        ctx.close()
        del layers, arena
        torch.cuda.empty_cache()


def stages():
    L, bs, H, D, NB, nblk = 32, 16, 8, 128, 4096, 2048
    ctx, layers, arena, U = setup(L, bs, H, D, NB, nblk)
    s = torch.cuda.Stream()
    nbytes = nblk * U
    for piece, st in [(16384, 4), (16384, 6), (16384, 8), (16384, 12), (32768, 2), (32768, 3), (32768, 4),
                      (32768, 6), (65536, 2), (65536, 3), (8192, 12), (8192, 24)]:
        for ctas in (148, 0):
            ctx.set_option(aqua.OPT_TMA_PIECE, piece)
            ctx.set_option(aqua.OPT_TMA_STAGES, st)
            ctx.set_option(aqua.OPT_MAX_CTAS, ctas)
            o, i = time_swaps(ctx, 10, s)
            print(json.dumps({"piece": piece, "stages": st, "max_ctas": ctas, "out_ms": round(o, 4),
                              "in_ms": round(i, 4), "out_hbm_GBps": round(2 * nbytes / o / 1e6, 1),
                              "in_hbm_GBps": round(2 * nbytes / i / 1e6, 1)}), flush=True)


def c5(host=False):
    L, H, D = 32, 8, 128
    for bs in (8, 16, 32, 64, 128):
        S = bs * H * D * 2
        U = 2 * L * S
        for nblk in (1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024):
            if nblk * U > (16 << 30) or (host and nblk * U > (4 << 30)):
                continue
            NB = 2 * nblk
            ctx, layers, arena, _ = setup(L, bs, H, D, NB, nblk, host=host)
            s = torch.cuda.Stream()
            reps = 20 if nblk * U < (1 << 30) else 5
            o, i = time_tickets(ctx, reps, s)
            print(json.dumps({"c5": "host" if host else "self", "bs": bs, "U": U, "blocks": nblk,
                              "bytes": nblk * U, "out_ms": round(o, 5), "in_ms": round(i, 5),
                              "out_GBps": round(nblk * U / o / 1e6, 2), "in_GBps": round(nblk * U / i / 1e6, 2)}),
                  flush=True)
            ctx.close()
            del layers, arena
            torch.cuda.empty_cache()


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "engines"
    if what == "engines":
        engines()
    elif what == "c5":
        c5(host=False)
    elif what == "c5host":
        c5(host=True)
    elif what == "stages":
        stages()
    elif what == "layers":
        layers()
    elif what == "prefix":
        prefix()
    elif what == "migrate":
        migrate()
    elif what == "tma_variants":
        tma_variants()
    elif what == "layer_overlap":
        layer_overlap()
    elif what == "duplex":
        duplex()
    elif what == "exchange":
        exchange()
    elif what == "torch_baseline":
        torch_baseline()
    elif what == "c5_multi":
        c5_multi()
    elif what == "ctas_stages":
        ctas_stages()
    elif what == "host_ctas":
        host_ctas()
    elif what == "self_ctas":
        self_ctas()
    elif what == "host_pcie":
        host_pcie()
    elif what == "tma_sched":
        tma_sched()
    elif what == "hybrid":
        hybrid()
    elif what == "small_chunks":
        small_chunks()
    elif what == "small_chunks2":
        small_chunks2()
    elif what == "small_ldst":
        small_ldst_sweep()
    elif what == "rate":
        rate()


def latency():
    """Host cost of one call (enqueue only), device time of one call on an
    idle GPU (ticket events), and back-to-back device time per call with the
    calls queued behind a sleep kernel (no host gaps).  AQUA_SWEEP_INLINE sets
    AQUA_OPT_INLINE_MAX (descriptors in the kernel parameters vs staged)."""
    import time
    inline = int(os.environ.get("AQUA_SWEEP_INLINE", "-1"))
    L, bs, H, D = 32, 16, 8, 128
    for nblk in (1, 8, 64, 256, 257, 1024, 2048, 4064, 4096):
        ctx, layers, arena, U = setup(L, bs, H, D, max(4096, 2 * nblk), nblk)
        if inline >= 0:
            ctx.set_option(aqua.OPT_INLINE_MAX, inline)
        s = torch.cuda.Stream()
        o, i = time_swaps(ctx, 20, s)
        ctx.set_option(aqua.OPT_TIMING, 1)
        dev = []
        for _ in range(20):
            t1 = ctx.swap_out([7], s.cuda_stream)
            _, t2 = ctx.swap_in([7], s.cuda_stream)
            torch.cuda.synchronize()
            dev.append((ctx.ticket_elapsed(t1), ctx.ticket_elapsed(t2)))
        ctx.set_option(aqua.OPT_TIMING, 0)
        enq = []
        for _ in range(50):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ctx.swap_out([7], s.cuda_stream)
            t1 = time.perf_counter()
            ctx.swap_in([7], s.cuda_stream)
            t2 = time.perf_counter()
            enq.append((t1 - t0, t2 - t1))
        torch.cuda.synchronize()
        q = []
        for _ in range(5):
            K = 20
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                torch.cuda._sleep(40_000_000)
            a.record(s)
            for _ in range(K):
                ctx.swap_out([7], s.cuda_stream)
                ctx.swap_in([7], s.cuda_stream)
            b.record(s)
            torch.cuda.synchronize()
            q.append(a.elapsed_time(b) / (2 * K))
        print(json.dumps({"latency": nblk, "bytes": nblk * U, "inline_max": ctx.get_option(aqua.OPT_INLINE_MAX),
                          "out_ms": round(o, 4), "in_ms": round(i, 4),
                          "ticket_out_ms": round(statistics.median(d[0] for d in dev), 4),
                          "ticket_in_ms": round(statistics.median(d[1] for d in dev), 4),
                          "queued_call_ms": round(statistics.median(q), 4),
                          "queued_GBps": round(nblk * U / statistics.median(q) / 1e6, 1),
                          "enqueue_out_us": round(1e6 * statistics.median(e[0] for e in enq), 1),
                          "enqueue_in_us": round(1e6 * statistics.median(e[1] for e in enq), 1)}), flush=True)
        ctx.close()
        del layers, arena
        torch.cuda.empty_cache()


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "latency":
    latency()


def small_calls():
    """Device time of 1..64-block calls (C2 shape, 2 MiB blocks) by engine
    and stage size, each measured behind a sleep kernel (no host gap), next
    to a 1-element torch kernel timed the same way (the launch + event floor)."""
    L, bs, H, D = 32, 16, 8, 128
    s = torch.cuda.Stream()
    x = torch.zeros(1, device="cuda")
    floor = []
    for _ in range(50):
        with torch.cuda.stream(s):
            torch.cuda._sleep(200_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            x.add_(1)
            b.record(s)
        torch.cuda.synchronize()
        floor.append(a.elapsed_time(b))
    print(json.dumps({"small_calls": "floor", "one_tiny_kernel_us": round(1e3 * statistics.median(floor), 2)}),
          flush=True)
    for nblk in (1, 2, 4, 8, 16, 64):
        ctx, layers, arena, U = setup(L, bs, H, D, 4096, nblk)
        for eng, piece in (("auto", 0), ("tma", 16384), ("tma", 8192), ("ldst", 0)):
            ctx.set_option(aqua.OPT_KERNEL, aqua.KERNEL_AUTO if eng == "auto" else ENG[eng])
            ctx.set_option(aqua.OPT_TMA_PIECE, piece)
            o, i = time_tickets(ctx, 30, s, sleep_cycles=200_000)
            ll = ctx.last_launch()
            print(json.dumps({"small_calls": nblk, "bytes": nblk * U, "engine": eng, "piece": piece,
                              "grid": ll["ctas"], "schedule": ll["schedule"],
                              "out_us": round(1e3 * o, 2), "in_us": round(1e3 * i, 2)}), flush=True)
        ctx.close()
        del layers, arena
        torch.cuda.empty_cache()


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "small_calls":
    small_calls()


def ncu_small():
    """For an ncu capture of the small-chunk kernel under AUTO: 1 GiB calls
    of S = AQUA_SWEEP_S (plane-major, L = 32, H = 1), 2 warm-up pairs then
    one swap_out + swap_in pair (launches 5 and 6)."""
    S = int(os.environ.get("AQUA_SWEEP_S", "512"))
    L, H, D = 32, 1, S // 32
    U = 2 * L * S
    nblk = (1 << 30) // U
    ctx, layers, arena, _ = setup(L, 16, H, D, 2 * nblk, nblk)
    s = torch.cuda.Stream()
    for _ in range(3):
        ctx.swap_out([7], s.cuda_stream)
        ctx.swap_in([7], s.cuda_stream)
    torch.cuda.synchronize()
    print(json.dumps({"ncu_small": S, "blocks": nblk, "launch": ctx.last_launch()}), flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "ncu_small":
    ncu_small()


def small_caps():
    """Sub-stage chunks under SM caps: AUTO (the hybrid ring + register warps)
    vs the small-chunk register kernel (512-thread CTAs when capped), device
    time per 1 GiB call behind a sleep kernel; S = AQUA_SWEEP_S, caps =
    AQUA_SWEEP_CAPS."""
    Ss = [int(x) for x in os.environ.get("AQUA_SWEEP_S", "512,1024,2048,4096,8192").split(",")]
    caps = [int(x) for x in os.environ.get("AQUA_SWEEP_CAPS", "8,16,32,64,96").split(",")]
    for S in Ss:
        L, H, D = 32, 1, S // 32
        U = 2 * L * S
        nblk = (1 << 30) // U
        ctx, layers, arena, _ = setup(L, 16, H, D, 2 * nblk, nblk)
        s = torch.cuda.Stream()
        for cap in caps:
            for eng in ("auto", "small"):
                ctx.set_option(aqua.OPT_KERNEL, aqua.KERNEL_AUTO if eng == "auto" else aqua.KERNEL_LDST)
                ctx.set_option(aqua.OPT_LDST_VARIANT, 3 if eng == "small" else 2)
                ctx.set_option(aqua.OPT_MAX_CTAS, cap)
                o, i = time_tickets(ctx, 5, s)
                ll = ctx.last_launch()
                print(json.dumps({"S": S, "cap": cap, "engine": eng, "kernel": ll["engine"], "variant": ll["variant"],
                                  "grid": ll["ctas"], "threads": ll["threads_per_cta"],
                                  "out_GBps_rw": round(2 * nblk * U / o / 1e6, 1),
                                  "in_GBps_rw": round(2 * nblk * U / i / 1e6, 1),
                                  "per_sm_rw": round(2 * nblk * U / ((o + i) / 2) / 1e6 / cap, 1)}), flush=True)
        ctx.close()
        del layers, arena
        torch.cuda.empty_cache()


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "small_caps":
    small_caps()



def block_order():
    """Does the order / locality of a prompt's blocks in the pool change the
    copy rate of small chunks?  One prompt of 1 GiB (plane-major, S =
    AQUA_SWEEP_S), AUTO, three block tables over the same pool: a random half
    of the blocks in random order (the sweeps' default: a fragmented pool),
    the same blocks sorted ascending, and one contiguous run.  Back-to-back
    (queued) and per-call (behind a sleep) device time."""
    Ss = [int(x) for x in os.environ.get("AQUA_SWEEP_S", "512,1024,2048,8192,32768").split(",")]
    for S in Ss:
        L = 32
        H, D = (1, S // 32) if S <= 4096 else (S // 4096, 128)
        U = 2 * L * S
        nblk = (1 << 30) // U
        NB = 2 * nblk
        layers = [torch.zeros(2 * NB * S, dtype=torch.uint8, device="cuda") for _ in range(L)]
        arena = torch.empty(nblk * U, dtype=torch.uint8, device="cuda")
        perm = block_permutation(NB, NB, seed=2).tolist()
        tables = {"random_half_random_order": perm[:nblk], "random_half_sorted": sorted(perm[:nblk]),
                  "contiguous": list(range(nblk))}
        s = torch.cuda.Stream()
        for name, bt in tables.items():
            ctx = aqua.Ctx(0, L, 16, H, D, 2, NB, [t.data_ptr() for t in layers])
            ctx.lend(0, arena.data_ptr(), nblk * U)
            rest = sorted(set(range(NB)) - set(bt))
            ctx.adopt_blocks(1, rest)
            ctx.adopt_blocks(7, bt)
            pair = time_queued(ctx, s, K=10, reps=3)
            o, i = time_tickets(ctx, 5, s)
            print(json.dumps({"S": S, "blocks": name, "nblk": nblk, "engine": ctx.last_launch()["engine"],
                              "queued_TBps_rw": round(4 * nblk * U / pair / 1e9, 3),
                              "per_call_out_TBps_rw": round(2 * nblk * U / o / 1e9, 3),
                              "per_call_in_TBps_rw": round(2 * nblk * U / i / 1e9, 3)}), flush=True)
            ctx.close()
        del layers, arena
        torch.cuda.empty_cache()


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "block_order":
    block_order()
