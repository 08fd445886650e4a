#!/usr/bin/env python3
"""bench.py -- preempt/resume KV paging on B200 (arXiv 2407.21255 hot path).

Default workload (BASELINE.json configs[1]): Llama-3-8B-shaped KV (32
layers, 8 KV heads, head_dim 128, bf16, block 16), one 32K-token prompt =
2048 blocks of U = 2 MiB (4 GiB) on a fragmented block table.  One step =
preempt (aqua_swap_out) + resume (aqua_swap_in) of that prompt: 2 x 4 GiB of
algorithmic bytes.  At N=1 the lender arena lives in the same GPU's HBM
("self-lender", HBM-bound); at N>1 (torchrun) rank r pages into HBM lent by
rank r^1 over NVLink (IPC handles exchanged once), every rank a borrower and
a lender (weak scaling; no collective on the data path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0 (contract in DESIGN.md "Measurement").
``--impl reference`` times the CPU oracle (the reference arm of this tier)
on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "KV swap GB/s per GPU pair vs 900 GB/s NVLink; preempt+resume latency/prompt"
# Bench workloads (BASELINE.json configs).  c2 = configs[1], the default and
# the one the metric is quoted on; c4 = one TP rank of configs[3] (Llama-3-70B
# KV over TP4: 2 KV heads per rank, S = 8 KiB), 32 prompts x 2048 tokens
# swapped in ONE batched call per direction.
CONFIGS = {
    "c2": dict(L=32, bs=16, H=8, D=128, e=2, NB=4096, nprompts=1, bpp=2048,
               desc="configs[1]: Llama-3-8B-shaped KV (L=32, H=8, D=128, bf16, block 16), one 32K-token prompt = "
                    "2048 blocks x 2 MiB on a fragmented block table"),
    "c4": dict(L=80, bs=16, H=2, D=128, e=2, NB=8192, nprompts=32, bpp=128,
               desc="configs[3] per rank: Llama-3-70B-shaped KV over TP4 (L=80, 2 KV heads, D=128, bf16, block 16), "
                    "32 prompts x 2048 tokens = 4096 blocks x 1.25 MiB, one batched call per direction"),
}
SHAPE = NB = NBLK = PIDS = CFG = None
SEED_PATTERN = 1234


def select_config(name):
    global SHAPE, NB, NBLK, PIDS, CFG
    CFG = dict(CONFIGS[name], name=name)
    SHAPE = {k: CFG[k] for k in ("L", "bs", "H", "D", "e")}
    NB = CFG["NB"]
    NBLK = CFG["nprompts"] * CFG["bpp"]
    PIDS = list(range(100, 100 + CFG["nprompts"]))


select_config("c2")


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, read+write bytes)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


NVLINK_MEASURED = 770.0   # GB/s per direction, peer copy (B200_PROFILING.md)
NVLINK_NOMINAL = 900.0    # GB/s per direction per GPU (NVLink 5), the north_star's denominator
RW_BOUND = 6820.0         # GB/s read + write: a copy on DRAM that time-shares 7.36 TB/s reads and 6.35 TB/s writes
# The paper's end-to-end results on 8x H100-80G, quoted as context only; the paper
# gives no swap GB/s or per-prompt swap latency for its own path.
PAPER_CONTEXT = {
    "ttft_under_burst": "20x lower than vLLM FCFS; 8x H100-80G, Llama-3.1-70B TP2, ShareGPT, 25 prompts then 2x rate "
                        "for 1 min (P:57, P:983-985)",
    "long_prompt_throughput": "4x vs FlexGen paging to DRAM (BASELINE.json says vLLM; the paper's baseline is FlexGen); "
                              "8x H100-80G, OPT-30B, 8192-token prompts (P:57, P:1009)",
    "a100_nvlink_copy": "50 GB/s at 4 MB, 200 GB/s at 64 MB, 2x A100-80GB (P:846-848)",
    "here_modelled": "MODELLED, not measured end to end: a responsiveness model of the C3 trace that puts each "
                     "measured swap time on the critical path of the virtual-clock schedule "
                     "(profiles/r01_c3_model_*.json) gives CFS a TTFT p50 28x below FCFS and, paging to the lender "
                     "instead of host DRAM, a TPOT p99 1.8x lower",
}


class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML during the timed region."""

    def __init__(self, index: int, period: float = 0.005):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": getattr(nv, "nvmlClocksEventReasonGpuIdle", 0x1),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": len(self.samples)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_oracle_sample(seconds: float = 10.0, nblk: int = 128):
    """The oracle as it stands (bytes mode, one host core) on a bounded sample
    of the same workload: a `nblk`-block prompt of the Llama-3-8B shape
    swapped out and back, repeated until `seconds` of CPU work."""
    import numpy as np
    from oracle import kvpool as kp
    from workloads import block_permutation, kv_random_bytes

    nb = 2 * nblk
    lay = kp.Layout(L=SHAPE["L"], bs=SHAPE["bs"], H=SHAPE["H"], D=SHAPE["D"], e=SHAPE["e"], NB=nb)
    layers = [kv_random_bytes(lay.layer_bytes, seed=l).copy() for l in range(lay.L)]
    pool = kp.Pool(lay, layers)
    pool.lend(kp.LOC_PEER, nblk * lay.U, np.zeros(nblk * lay.U, np.uint8))
    pool.adopt_blocks(7, block_permutation(nb, nblk, seed=2).tolist())
    reps, t_work = 0, 0.0
    t_end = time.perf_counter() + seconds
    while time.perf_counter() < t_end or reps == 0:
        t0 = time.perf_counter()
        pool.swap_out([7])
        pool.swap_in([7])
        t_work += time.perf_counter() - t0
        reps += 1
    moved = reps * 2 * nblk * lay.U
    # host context: one core's plain memcpy rate, same bytes definition
    a, b = np.ones(256 << 20, np.uint8), np.empty(256 << 20, np.uint8)
    np.copyto(b, a)
    mt = []
    for _ in range(5):
        t0 = time.perf_counter()
        np.copyto(b, a)
        mt.append(time.perf_counter() - t0)
    memcpy = a.nbytes / sorted(mt)[2] / 1e9
    return {"value": moved / t_work / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
            "host_memcpy_1core_GBps": round(memcpy, 2),
            "sample": f"{reps} x (swap_out + swap_in) of a {nblk}-block prompt (U={lay.U / 2**20:g} MiB, "
                      f"{nblk * lay.U / 2**20:.0f} MiB per direction) of the {CFG['name']} shape, "
                      f"numpy bytes mode, {t_work:.1f} s", "seconds_per_step": t_work / reps,
            "bytes_per_step": 2 * nblk * lay.U}


def run_reference(args):
    """The reference arm of this tier: the CPU oracle, as it stands."""
    ws, rank, _ = _dist()
    if ws > 1 and rank != 0:
        return
    import numpy as np
    from oracle import kvpool as kp
    from workloads import block_permutation, kv_random_bytes
    nblk = 128
    nb = 2 * nblk
    lay = kp.Layout(L=SHAPE["L"], bs=SHAPE["bs"], H=SHAPE["H"], D=SHAPE["D"], e=SHAPE["e"], NB=nb)
    pool = kp.Pool(lay, [kv_random_bytes(lay.layer_bytes, seed=l).copy() for l in range(lay.L)])
    pool.lend(kp.LOC_PEER, nblk * lay.U, np.zeros(nblk * lay.U, np.uint8))
    pool.adopt_blocks(7, block_permutation(nb, nblk, seed=2).tolist())
    for _ in range(args.warmup):
        pool.swap_out([7])
        pool.swap_in([7])
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        pool.swap_out([7])
        pool.swap_in([7])
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    moved = args.steps * 2 * nblk * lay.U
    val = moved / tot / 1e9
    sample = (f"each step = swap_out + swap_in of a {nblk}-block prompt ({nblk * lay.U / 2**20:.0f} MiB per "
              f"direction) of the {CFG['name']} shape (U = {lay.U / 2**20:g} MiB per block), oracle bytes mode, 1 core")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * tot / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": _config(args, reference=True, n=args.gpus, roles=args.roles),
        "sample": f"each timed step moves a {nblk}-block sample ({nblk}/{NBLK} of the config's {NBLK} blocks per "
                  f"direction); value is GB/s over the sample's bytes, so it compares with our arm's GB/s",
        "cpu_baseline": {"value": round(val, 3), "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": round(val, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _config(args, reference=False, n=1, roles="both"):
    U = 2 * SHAPE["L"] * SHAPE["bs"] * SHAPE["H"] * SHAPE["D"] * SHAPE["e"]
    if n == 1:
        how, lending = "(self-lender: arena in the same HBM)", "self (same HBM)"
    elif roles == "split":
        how = f"(ranks 0..{n // 2 - 1} page into HBM lent by ranks {n // 2}..{n - 1} over NVLink)"
        lending = f"split roles: {n // 2} borrowers -> {n // 2} lenders over NVLink"
    else:
        how, lending = "(peer lender = partner rank over NVLink)", f"pairs over NVLink ({n} ranks, each both roles)"
    return {"workload": CFG["desc"] + "; step = preempt + resume " + how,
            "name": CFG["name"], "prompts": CFG["nprompts"], "tokens_per_prompt": CFG["bpp"] * SHAPE["bs"],
            "layout": dict(SHAPE, NB=NB), "lending": lending,
            "engine": args.engine, "bytes_per_step": 2 * NBLK * U,
            "l2": f"inputs ({NBLK * U / 2**30:.1f} GiB per direction) >> 126 MB L2; no flush needed"}


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2407_21255_b200 import aqua
    from workloads import block_permutation

    ws, rank, local = _dist()
    shared = os.environ.get("AQUA_BENCH_SHARED_GPU") == "1"   # test mode: all ranks on cuda:0, gloo
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    L, bs, H, D, e = SHAPE["L"], SHAPE["bs"], SHAPE["H"], SHAPE["D"], SHAPE["e"]
    S = bs * H * D * e
    U = 2 * L * S
    layer_bytes = 2 * NB * S
    layers = [torch.zeros(layer_bytes, dtype=torch.uint8, device=dev) for _ in range(L)]
    ctx = aqua.Ctx(local, L, bs, H, D, e, NB, [t.data_ptr() for t in layers])
    if args.engine != "auto":
        ctx.set_option(aqua.OPT_KERNEL, {"tma": aqua.KERNEL_TMA, "ldst": aqua.KERNEL_LDST,
                                         "per_chunk": aqua.BASE_PER_CHUNK,
                                         "gather_temp": aqua.BASE_GATHER_TEMP}[args.engine])
    if args.max_ctas:
        ctx.set_option(aqua.OPT_MAX_CTAS, args.max_ctas)
    if args.piece:
        ctx.set_option(aqua.OPT_TMA_PIECE, args.piece)
    if args.inline_max >= 0:
        ctx.set_option(aqua.OPT_INLINE_MAX, args.inline_max)

    arena_bytes = NBLK * U
    ipc_ptr = imported = None
    matching = None
    borrower = True                  # this rank pages its own prompts (every rank unless --roles split)
    roles = args.roles if ws > 1 else "both"
    topology = None
    if ws == 1:
        arena = torch.empty(arena_bytes, dtype=torch.uint8, device=dev)
        ctx.lend(local, arena.data_ptr(), arena_bytes)
        mode = "self-lender"
    else:
        from paper_2407_21255_b200.pairing import best_bipartite, best_matching, exchange, measure_p2p
        # pairing from the measured topology: rank 0's P2P
        # bandwidth matrix (default), or P2P reachability rows from every
        # rank (--no-measure-topology, and the shared-GPU test mode); then
        # the max-min perfect matching (roles "both") or the max-min
        # borrower -> lender assignment (roles "split", configs[3])
        if args.measure_topology and not shared:
            bw = measure_p2p(ws) if rank == 0 else None
            bw = exchange(bw)[0]
            topology = "measured P2P copy GB/s (pairing.measure_p2p)"
        else:
            row = [0.0 if j == local else (1.0 if shared or aqua.can_access_peer(local, j) else 0.0)
                   for j in range(ws)]
            bw = exchange(row)
            topology = "P2P reachability"
        if roles == "split":
            if ws % 2:
                raise SystemExit("--roles split needs an even number of GPUs")
            half = ws // 2
            matching = best_bipartite(bw, list(range(half)), list(range(half, ws)))
            borrower = rank < half
        else:
            matching = best_matching(bw)
        partner = matching[rank]
        lends = roles == "both" or not borrower
        if lends:
            ipc_ptr = aqua.ipc_alloc(local, arena_bytes)      # what this rank lends to its partner
        handles = exchange((rank, local, aqua.ipc_export(ipc_ptr) if lends else None))
        if not borrower:
            mode = f"lender for rank{partner}"
        elif partner == rank:
            ctx.lend(local, ipc_ptr, arena_bytes)
            mode = "self-lender"
        else:
            try:
                imported = aqua.ipc_import(local, handles[partner][2])
                ctx.lend(aqua.MAPPED, imported, arena_bytes)
                mode = f"peer-lender rank{partner}"
            except aqua.AquaError as err:        # no P2P path to the partner: page into our own HBM
                imported = None                  # (a fresh arena: the partner may still write into ipc_ptr)
                arena = torch.empty(arena_bytes, dtype=torch.uint8, device=dev)
                ctx.lend(local, arena.data_ptr(), arena_bytes)
                mode = f"self-lender (peer rank{partner} unreachable: {err})"
    bpp = CFG["bpp"]
    if borrower:
        perm = block_permutation(NB, NB, seed=2).tolist()
        ctx.adopt_blocks(1, perm[NBLK:])      # filler: keeps the prompts' blocks scattered over the pool
        for i, pid in enumerate(PIDS):
            ctx.adopt_blocks(pid, perm[i * bpp:(i + 1) * bpp])
            ctx.kv_fill_pattern(pid, 0, bpp * bs, SEED_PATTERN)
    torch.cuda.synchronize()
    swap = torch.cuda.Stream(device=dev)
    sw = swap.cuda_stream

    if borrower:
        for _ in range(args.warmup):
            ctx.swap_out(PIDS, sw)
            ctx.swap_in(PIDS, sw)
    torch.cuda.synchronize()

    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    n0 = ctx.launch_count()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record(swap)
        for k in range(K if borrower else 0):
            ev[k][0].record(swap)
            ctx.swap_out(PIDS, sw)
            ev[k][1].record(swap)
            ctx.swap_in(PIDS, sw)
            ev[k][2].record(swap)
        end.record(swap)
        torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    launches = ctx.launch_count() - n0
    try:
        shape = ctx.last_launch()          # what the library's AUTO policy launched (the swap_in of the last step)
    except aqua.AquaError:                 # a baseline engine (or a lender rank) that launched no kernel of ours
        shape = {"engine": args.engine}
    total_ms = start.elapsed_time(end) if borrower else 0.0
    out_ms = [a.elapsed_time(b) for a, b, _ in ev] if borrower else [0.0]
    in_ms = [b.elapsed_time(c) for _, b, c in ev] if borrower else [0.0]
    t = torch.tensor([total_ms], device="cpu" if shared else dev, dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms_max = float(t.item())

    # parity at full size: the resumed prompt still holds its pattern
    mism = 0
    if borrower:
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        for pid in PIDS:
            ctx.kv_verify_pattern(pid, bpp * bs, SEED_PATTERN, cnt.data_ptr())
        torch.cuda.synchronize()
        mism = int(cnt.item())
    if mism:
        raise SystemExit(f"rank {rank}: {mism} KV words differ after preempt/resume -- parity failure")

    # end to end through the public API: host pid list in; descriptor uploads
    # inside; the new block table goes host -> device (pinned) for the decode
    # kernels; a 16-byte probe of each resumed prompt's first K chunk comes
    # back device -> host; host-synchronised every step
    S0 = SHAPE["bs"] * SHAPE["H"] * SHAPE["D"] * SHAPE["e"]
    e2e_t, lat_out, lat_in = [0.0], [0.0], [0.0]
    if borrower:
        bt_h = torch.empty(NBLK, dtype=torch.int32, pin_memory=True)
        bt_d = torch.empty(NBLK, dtype=torch.int32, device=dev)
        probe_h = torch.empty(len(PIDS), 16, dtype=torch.uint8, pin_memory=True)

        def first_chunk(pid):
            b = ctx.query(pid, with_ids=True)[3][0]
            return layers[0][b * S0:b * S0 + 16]

        probe_ref = torch.stack([first_chunk(pid).cpu() for pid in PIDS])
        e2e_t, lat_out, lat_in = [], [], []
        reps = max(20, min(K, 50))
        for _ in range(reps):           # per-call host latency: sync on each ticket
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ctx.sync(ctx.swap_out(PIDS, sw))
            t1 = time.perf_counter()
            ctx.sync(ctx.swap_in(PIDS, sw)[1])
            t2 = time.perf_counter()
            lat_out.append(t1 - t0)
            lat_in.append(t2 - t1)
        # the probes: one 16-byte copy for a single prompt; with several, their row indices go up in
        # one pinned H2D copy, one gather on the device, and ONE D2H copy of 16 bytes per prompt
        rows0 = layers[0].view(-1, 16)                  # 16-byte rows of layer 0
        bt_np = bt_h.numpy()
        idx_h = torch.empty(len(PIDS), dtype=torch.int64, pin_memory=True)
        idx_d = torch.empty(len(PIDS), dtype=torch.int64, device=dev)
        idx_np = idx_h.numpy()
        for _ in range(reps):           # the step as a user runs it: no sync between the calls
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ctx.swap_out(PIDS, sw)
            new, _ = ctx.swap_in(PIDS, sw, as_arrays=True)
            with torch.cuda.stream(swap):
                if len(new) == 1:
                    bt_np[:] = new[0]
                    b = int(new[0][0])
                    probe_h[0].copy_(layers[0][b * S0:b * S0 + 16], non_blocking=True)
                else:
                    bt_np[:] = np.concatenate(new)
                    idx_np[:] = [int(ids[0]) * (S0 // 16) for ids in new]
                    idx_d.copy_(idx_h, non_blocking=True)
                    probe_h.copy_(rows0.index_select(0, idx_d), non_blocking=True)
                bt_d.copy_(bt_h, non_blocking=True)
            swap.synchronize()
            e2e_t.append(time.perf_counter() - t0)
        if not torch.equal(probe_h, probe_ref):
            raise SystemExit(f"rank {rank}: e2e probe of the resumed KV differs -- parity failure")

    bytes_per_step = 2 * NBLK * U
    n_borrowers = ws if roles == "both" else ws // 2
    value = n_borrowers * K * bytes_per_step / (total_ms_max / 1e3) / 1e9
    out_avg, in_avg = statistics.mean(out_ms), statistics.mean(in_ms)
    per_rank = None
    if ws > 1:                        # every rank's own per-direction link rate and preempt+resume latency
        from paper_2407_21255_b200.pairing import exchange
        per_rank = []
        for r, m, b, o, i, lo, li, e2 in exchange((rank, mode, borrower, out_avg, in_avg,
                                                   statistics.median(lat_out), statistics.median(lat_in),
                                                   statistics.median(e2e_t))):
            rec = {"rank": r, "mode": m}
            if b:
                rec.update({"swap_out_GBps": round(NBLK * U / (o / 1e3) / 1e9, 1),
                            "swap_in_GBps": round(NBLK * U / (i / 1e3) / 1e9, 1),
                            "preempt_device_ms": round(o, 4), "resume_device_ms": round(i, 4),
                            "preempt_resume_device_ms": round(o + i, 4),
                            "preempt_resume_host_p50_ms": round(1e3 * (lo + li), 4),
                            "e2e_step_p50_ms": round(1e3 * e2, 4)})
            per_rank.append(rec)

    host = None
    if ws == 1 and not args.no_host_baselines and CFG["name"] == "c2":
        host = host_baselines(ctx, layers, dev, aqua, args)

    if rank != 0:
        _cleanup(aqua, local, ipc_ptr, imported, ws)
        return
    hbm_peak, hbm_src = _peaks()
    north = None
    if ws == 1:
        ach = 2 * NBLK * U / (out_avg / 1e3) / 1e9           # read + write bytes, same HBM
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(ach / hbm_peak, 4), "traffic": _ncu_traffic(CFG["name"]),
                "kernel": "swap_tma_kernel<kOut> (swap_out launch)" if args.engine in ("auto", "tma")
                else f"{args.engine} swap_out", "peak_source": hbm_src,
                "algorithmic_bytes_per_launch": 2 * NBLK * U,
                "swap_in_achieved": round(2 * NBLK * U / (in_avg / 1e3) / 1e9, 1),
                "ncu": _ncu_record() if CFG["name"] == "c2" else None,
                "rw_bound": {"value": RW_BOUND, "frac": round(ach / RW_BOUND, 4),
                             "basis": "DRAM time-shared between reads and writes: 2 / (1/7.36 + 1/6.35) TB/s, pure "
                                      "read / pure write probe on this B200 (profiles/r01_hbm_probe.jsonl)"}}
        north = {"per_pair_per_direction_GBps": {"swap_out": round(NBLK * U / (out_avg / 1e3) / 1e9, 1),
                                                 "swap_in": round(NBLK * U / (in_avg / 1e3) / 1e9, 1)},
                 "link": "none: at N=1 the lender is the same GPU's HBM (the north_star's '1 GPU (local/host)'); "
                         "the 900 GB/s NVLink target applies from N=2"}
    else:
        peers = [p for p in per_rank if "swap_out_GBps" in p]
        lo_out = min(p["swap_out_GBps"] for p in peers)
        lo_in = min(p["swap_in_GBps"] for p in peers)
        ach = NBLK * U / (out_avg / 1e3) / 1e9                # rank 0's bytes across the link per direction
        roof = {"bound": "nvlink", "achieved": round(ach, 1), "peak": NVLINK_MEASURED, "unit": "GB/s",
                "frac": round(ach / NVLINK_MEASURED, 4), "traffic": None,
                "peak_source": "fallback: measured peer copy per direction (B200_PROFILING.md), "
                               "MEASURED_PEAKS.json has no NVLink figure",
                "nominal_peak": NVLINK_NOMINAL, "frac_of_nominal": round(ach / NVLINK_NOMINAL, 4),
                "kernel": "swap_out launch (rank 0)", "algorithmic_bytes_per_launch": NBLK * U,
                "swap_in_achieved": round(NBLK * U / (in_avg / 1e3) / 1e9, 1),
                "traffic_note": "NVLink bytes need ncu --replay-mode application on a 2-GPU box "
                                "(scripts/gpu_runs/r02_nvlink_ncu.sh); not captured yet"}
        north = {"per_pair_per_direction_GBps": {"swap_out_min_over_pairs": lo_out, "swap_in_min_over_pairs": lo_in},
                 "frac_of_900": {"swap_out": round(lo_out / NVLINK_NOMINAL, 4),
                                 "swap_in": round(lo_in / NVLINK_NOMINAL, 4)},
                 "frac_of_770_measured": {"swap_out": round(lo_out / NVLINK_MEASURED, 4),
                                          "swap_in": round(lo_in / NVLINK_MEASURED, 4)},
                 "target": ">= 0.8 of 900 GB/s per direction per GPU pair (BASELINE.json north_star)",
                 "pairs": n_borrowers, "roles": roles, "topology": topology}
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_oracle_sample(args.cpu_seconds)
        cpu.pop("seconds_per_step")
        cpu.pop("bytes_per_step")
        cpu["value"] = round(cpu["value"], 3)
    e2e_val = n_borrowers * bytes_per_step / statistics.median(e2e_t) / 1e9
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": ws, "steps": K,
        "warmup": args.warmup, "ms_per_step": round(total_ms_max / K, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": _config(args, n=ws, roles=roles),
        "mode": mode,
        "pairing": matching,
        "per_rank": per_rank,
        "north_star": north,
        "preempt_resume_ms": {"preempt_device_ms": round(out_avg, 4), "resume_device_ms": round(in_avg, 4),
                              "sum_device_ms": round(out_avg + in_avg, 4),
                              "prompts_per_call": len(PIDS),
                              "per_prompt_sum_device_ms": round((out_avg + in_avg) / len(PIDS), 4),
                              "preempt_host_p50_ms": round(1e3 * statistics.median(lat_out), 4),
                              "resume_host_p50_ms": round(1e3 * statistics.median(lat_in), 4),
                              "sum_host_p50_ms": round(1e3 * (statistics.median(lat_out) +
                                                               statistics.median(lat_in)), 4),
                              "e2e_step_p50_ms": round(1e3 * statistics.median(e2e_t), 4),
                              "preempt_host_p99_ms": round(1e3 * _pct(lat_out, 0.99), 4),
                              "resume_host_p99_ms": round(1e3 * _pct(lat_in, 0.99), 4),
                              "what": "device = CUDA events on the swap stream around each call; host = wall time from "
                                      "the C-ABI call to its ticket completing (aqua_sync); a call carries every "
                                      "prompt of the config, per-prompt = whole call / prompts (equal prompt sizes, "
                                      "so the byte-weighted attribution is the plain share)"},
        "launch_ms": {"swap_out": {q: round(_pct(out_ms, v), 4) for q, v in (("p10", .1), ("p50", .5), ("p90", .9))},
                      "swap_in": {q: round(_pct(in_ms, v), 4) for q, v in (("p10", .1), ("p50", .5), ("p90", .9))}},
        "launch_shape": dict(shape, blocks_per_launch=NBLK, block_tokens=SHAPE["bs"],
                             chunk_bytes=SHAPE["bs"] * SHAPE["H"] * SHAPE["D"] * SHAPE["e"], block_bytes_U=U),
        "host": _host_info(),
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": {"value": round(e2e_val, 2), "unit": "GB/s",
                "h2d_bytes_per_step": 2 * NBLK * 8 + NBLK * 4 + (8 * len(PIDS) if len(PIDS) > 1 else 0),
                "d2h_bytes_per_step": 16 * len(PIDS),
                "what": "aqua_swap_out + aqua_swap_in through the C ABI from host pid lists, host bookkeeping and "
                        "descriptor H2D upload (8 B per block per call), both calls queued back to back, then the new block table H2D from pinned "
                        "memory (4 B per block) and a 16-byte D2H probe of each resumed prompt's first K chunk "
                        "(checked against its pre-swap value; with several prompts their row indices go up in one "
                        "8 B-per-prompt H2D copy and the probes come back in one gathered D2H copy), "
                        "host-synchronised every step; the KV stays device-resident"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "parity": f"pattern verify: {mism} mismatching words over all {len(PIDS)} prompt(s) "
                  f"({NBLK * SHAPE['bs']} tokens) after {args.warmup + K} preempt/resume cycles",
        "host_baseline": host,
        "preempt_resume_vs_host": (round(host["best_preempt_resume_ms"] / (out_avg + in_avg), 1) if host else None),
        "paper_context": PAPER_CONTEXT,
    }
    print(json.dumps(line), flush=True)
    _cleanup(aqua, local, ipc_ptr, imported, ws)


def _pct(xs, q):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(q * len(xs)))]


def _sm_count():
    import torch
    return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count


def _host_info():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def _cleanup(aqua, local, ipc_ptr, imported, ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        if imported:
            aqua.ipc_close(local, imported)
        dist.barrier()
        if ipc_ptr:
            aqua.ipc_free(local, ipc_ptr)
        dist.destroy_process_group()


def _ncu_summary():
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return None
    return None


def _ncu_traffic(config="c2"):
    """dram__bytes_read.sum + dram__bytes_write.sum of one swap_out launch of
    this configuration in the committed capture (None if not captured)."""
    d = _ncu_summary()
    if not d:
        return None
    if config == "c2":
        return d.get("swap_out_traffic_bytes")
    return (d.get(f"{config}_swap_out") or {}).get("traffic_B")


def _ncu_record():
    """The committed ncu capture of this kernel (SURVEY 8(d) report record:
    achieved DRAM rate from the profiler, beside the event-timed one)."""
    d = _ncu_summary()
    if not d or "swap_out" not in d:
        return None
    o = d["swap_out"]
    return {"dram_TBps": round(o.get("dram_TBps", 0.0), 3),
            "pct_of_theoretical_dram": round(o.get("gpu_dram_throughput_pct_of_theoretical", 0.0), 1),
            "gpu_time_ms": round(o.get("gpu_time_ms", 0.0), 4), "source": "profiles/ncu_summary.json"}


def host_baselines(ctx_dev, layers, dev, aqua, args):
    """The paper's DRAM baseline: the same prompt
    paged to pinned host memory over PCIe with every copy engine; plus the
    plain PCIe copy peak.  Best-of is the comparator for the 32K prompt."""
    import torch
    L, bs, H, D, e = SHAPE["L"], SHAPE["bs"], SHAPE["H"], SHAPE["D"], SHAPE["e"]
    U = 2 * L * bs * H * D * e
    ctx = aqua.Ctx(dev.index, L, bs, H, D, e, NB, [t.data_ptr() for t in layers])
    ctx.lend(aqua.HOST, 0, NBLK * U)
    ctx.adopt_blocks(8, list(range(NBLK)))          # filler: resumes land back on 2048..4095
    ctx.adopt_blocks(9, list(range(NBLK, 2 * NBLK)))
    s = torch.cuda.Stream(device=dev)
    res = {}
    for name, eng in (("tma_zero_copy", aqua.KERNEL_TMA), ("ldst_zero_copy", aqua.KERNEL_LDST),
                      ("ce_host_staged", aqua.KERNEL_CE_HOST),
                      ("per_chunk_memcpy", aqua.BASE_PER_CHUNK), ("gather_temp_memcpy", aqua.BASE_GATHER_TEMP)):
        ctx.set_option(aqua.OPT_KERNEL, eng)
        try:
            ctx.swap_out([9], s.cuda_stream)
            ctx.swap_in([9], s.cuda_stream)
            torch.cuda.synchronize()
            outs, ins = [], []
            for _ in range(args.host_reps):
                a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                a.record(s)
                ctx.swap_out([9], s.cuda_stream)
                b.record(s)
                ctx.swap_in([9], s.cuda_stream)
                c.record(s)
                torch.cuda.synchronize()
                outs.append(a.elapsed_time(b))
                ins.append(b.elapsed_time(c))
            res[name] = {"out_GBps": round(NBLK * U / (min(outs) / 1e3) / 1e9, 2),
                         "in_GBps": round(NBLK * U / (min(ins) / 1e3) / 1e9, 2),
                         "preempt_resume_ms": round(min(outs) + min(ins), 3)}
        except Exception as ex:  # a baseline that cannot run is reported, not fatal
            res[name] = {"error": str(ex)[:200]}
    ctx.close()
    # raw PCIe: 1 GiB pinned copies each way
    h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    d.copy_(h)
    torch.cuda.synchronize()
    best = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        ts = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        best[name] = round((1 << 30) / (min(ts) / 1e3) / 1e9, 2)
    ok = {k: v for k, v in res.items() if "preempt_resume_ms" in v}
    bestk = min(ok, key=lambda k: ok[k]["preempt_resume_ms"]) if ok else None
    return {"variants": res, "pcie_copy_GBps": best, "best": bestk,
            "best_preempt_resume_ms": ok[bestk]["preempt_resume_ms"] if bestk else None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--engine", default="auto", choices=["auto", "tma", "ldst", "per_chunk", "gather_temp"])
    ap.add_argument("--max-ctas", type=int, default=0)
    ap.add_argument("--piece", type=int, default=0)
    ap.add_argument("--inline-max", type=int, default=-1,
                    help="AQUA_OPT_INLINE_MAX: largest call whose descriptors ride in the kernel parameters")
    ap.add_argument("--no-host-baselines", action="store_true")
    ap.add_argument("--host-reps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--measure-topology", action=argparse.BooleanOptionalAction, default=True,
                    help="N>1: pair GPUs by rank 0's measured P2P bandwidth matrix (default); "
                         "--no-measure-topology pairs by P2P reachability")
    ap.add_argument("--roles", choices=["both", "split"], default="both",
                    help="N>1: 'both' = every rank a borrower and a lender (bidirectional pairs); 'split' = ranks "
                         "0..N/2-1 borrow from ranks N/2..N-1 (configs[3]: 4 borrowers -> 4 lenders)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    select_config(args.config)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
