"""C3 (BASELINE configs[2]) on the GPU: the bursty trace through the native
CFS scheduler + libaqua paging + a synthetic decode, 1 borrower + 1 lender.

    python scripts/c3_run.py --policy cfs-peer|cfs-host|fcfs [--proxy-gb G] [--check-oracle]

At N=1 the "peer" lender arena lives in the same GPU (self-lender); the
decode writes each new token's closed-form KV pattern (C-11) on a decode
stream, swaps run on a swap stream, and every resumed prompt is verified
against the pattern right after its swap_in (restore invariant at full
scale).  --check-oracle also replays the oracle's metadata-mode run and
requires an identical call log.  Prints one JSON line.
"""
import argparse
import json
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2407_21255_b200 import aqua  # noqa: E402
from paper_2407_21255_b200.cfs import POLICY_CFS, POLICY_FCFS, Scheduler  # noqa: E402
from paper_2407_21255_b200.driver import run_trace  # noqa: E402
from workloads import burst_trace  # noqa: E402

NB = 4152          # scripts/c3_nb.py
L, bs, H, D, e = 32, 16, 8, 128, 2
SEED = 77


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--policy", default="cfs-peer", choices=["cfs-peer", "cfs-host", "fcfs"])
    ap.add_argument("--proxy-gb", type=float, default=0.0, help="decode proxy: GB of HBM streamed per iteration")
    ap.add_argument("--lender-gib", type=int, default=64)
    ap.add_argument("--host-gib", type=int, default=64)
    ap.add_argument("--check-oracle", action="store_true")
    ap.add_argument("--serial", action="store_true", help="swaps on the decode stream (no overlap), for A8")
    ap.add_argument("--exchange", action="store_true", help="reschedules with both lists use aqua_swap_exchange")
    ap.add_argument("--native", action="store_true", help="run the loop in C++ (aqua_trace_run)")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--trace-seed", type=int, default=1, help="seed of the bursty trace (BASELINE configs[2]: 1)")
    ap.add_argument("--elastic", default="", help="t_reclaim,t_relend (virtual s): NEXT-1 lender reclaim + FCFS "
                                                   "fallback, then re-offer")
    args = ap.parse_args()

    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    shared = os.environ.get("AQUA_BENCH_SHARED_GPU") == "1"
    devi = 0 if (ws == 1 or shared) else rank
    dev = torch.device("cuda", devi)
    torch.cuda.set_device(devi)
    S = bs * H * D * e
    U = 2 * L * S
    lend_bytes = args.lender_gib << 30
    if ws == 2:
        # 1 borrower (rank 0) + 1 lender (rank 1, another process -- another
        # GPU, or the same one with AQUA_BENCH_SHARED_GPU=1): the lender offers
        # HBM through a CUDA IPC handle; no data-path collective
        import torch.distributed as dist
        from paper_2407_21255_b200.pairing import exchange
        dist.init_process_group("gloo")
        if rank == 1:
            ptr = aqua.ipc_alloc(devi, lend_bytes)
            exchange((aqua.ipc_export(ptr), lend_bytes))
            dist.barrier()                    # the borrower runs the trace
            dist.barrier()                    # ... and has closed its mapping
            aqua.ipc_free(devi, ptr)
            dist.destroy_process_group()
            return
        handle = exchange(None)[1][0]
    layers = [torch.zeros(2 * NB * S, dtype=torch.uint8, device=dev) for _ in range(L)]
    ctx = aqua.Ctx(devi, L, bs, H, D, e, NB, [t.data_ptr() for t in layers])
    arena = None
    lend_dev, lend_ptr = devi, 0
    if args.policy == "cfs-peer":
        if ws == 2:
            lend_dev, lend_ptr = aqua.MAPPED, aqua.ipc_import(devi, handle)
        else:
            arena = torch.empty(lend_bytes, dtype=torch.uint8, device=dev)
            lend_ptr = arena.data_ptr()
        ctx.lend(lend_dev, lend_ptr, lend_bytes)
    ctx.lend(aqua.HOST, 0, args.host_gib << 30)
    ctx.set_option(aqua.OPT_TIMING, 1)               # per-swap device time via aqua_ticket_elapsed
    pol = POLICY_FCFS if args.policy == "fcfs" else POLICY_CFS
    sched = Scheduler(NB=NB, bs=bs, b=512, k=8, policy=pol)
    trace = burst_trace(seed=args.trace_seed)
    dec = torch.cuda.Stream(device=dev)
    swp = dec if args.serial else torch.cuda.Stream(device=dev)
    swp2 = torch.cuda.Stream(device=dev) if args.exchange else None
    mism = torch.zeros(1, dtype=torch.int64, device=dev)
    written = {}          # pid -> KV tokens written so far
    swap_events = []      # (kind, nblocks, ticket, npids, iteration)
    proxy = None
    if args.proxy_gb > 0:
        proxy = torch.empty(int(args.proxy_gb * 1e9) // 8, dtype=torch.int64, device=dev)
        proxy_out = torch.empty((), dtype=torch.int64, device=dev)

    def stream_sync(kind, ticket):
        if kind == "before_swap_out":
            swp.wait_stream(dec)                      # the blocks' last writer is the decode
        elif kind == "after_swap_in":
            ctx.wait(ticket, dec.cuda_stream)         # decode waits only for what it needs

    def on_swap(kind, pids, ticket, n):
        swap_events.append((kind, n, ticket, len(pids), iters["n"]))
        if kind == "in" and not args.no_verify:
            for p in pids:
                ctx.kv_verify_pattern(p, written.get(p, 0), SEED, mism.data_ptr(), dec.cuda_stream)

    iters = {"n": 0}
    plen = {rid: (P, O) for rid, _, P, O in trace}
    arrival = {rid: a for rid, a, _, _ in trace}
    gen = {}
    first_it, last_it = {}, {}
    it_tokens = []

    v_start = []

    def on_iteration(i, work):
        it_tokens.append(sum(w[2] for w in work))
        v_start.append(sched.vclock())
        for pid, ctx0, tok, grow, phase in work:
            written[pid] = ctx0 + tok
            P, O = plen[pid]
            if phase == 0 and ctx0 + tok == P:
                first_it[pid] = i
                gen[pid] = 1
            elif phase == 1:
                gen[pid] += 1
            if gen.get(pid, 0) >= O:
                last_it[pid] = i
        if proxy is not None:
            with torch.cuda.stream(dec):
                torch.sum(proxy, dim=0, out=proxy_out)
        iters["n"] += 1

    torch.cuda.synchronize()
    n0 = ctx.launch_count()
    t0 = time.perf_counter()
    elastic = None
    if args.elastic:
        tr_, tl_ = (float(x) for x in args.elastic.split(","))
        elastic = {"t_reclaim": tr_, "t_relend": tl_, "relend": (lend_dev, lend_ptr, lend_bytes)}
    if args.native:
        from paper_2407_21255_b200.cfs import run_trace_native
        if elastic or args.proxy_gb:
            raise SystemExit("--native runs the plain trace (no elastic events, no decode proxy)")
        log, st = run_trace_native(trace, ctx, sched, decode_stream=dec.cuda_stream, swap_stream=swp.cuda_stream,
                                   swap_stream2=swp2.cuda_stream if swp2 is not None else 0, fill_seed=SEED,
                                   d_mismatches=0 if args.no_verify else mism.data_ptr(),
                                   record_log=args.check_oracle)
        st["swap_calls"] = []
    else:
        log, st = run_trace(trace, ctx, sched, fill_seed=SEED, decode_stream=dec.cuda_stream,
                            swap_stream=swp.cuda_stream, on_iteration=on_iteration, stream_sync=stream_sync,
                            on_swap=on_swap, record_log=args.check_oracle, elastic=elastic,
                            exchange_stream=swp2.cuda_stream if swp2 is not None else None)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    launches = ctx.launch_count() - n0
    # per-call device time of the copies (library timing events)
    per_block_ms = []
    dev_ms = {"out": 0.0, "in": 0.0}
    swap_ms_at = [0.0] * (len(it_tokens) + 1)
    by_iter = {}
    for kind, n, tk, npids, at in swap_events:
        if n == 0:
            continue
        ms = ctx.ticket_elapsed(tk)
        dev_ms[kind] += ms
        per_block_ms.append((kind, ms, n, npids))
        by_iter.setdefault(at, []).append(ms)
    for at, mss in by_iter.items():
        # an exchange runs its two directions concurrently: its critical path
        # is the longer one; separate calls are sequential on the swap stream
        swap_ms_at[at] = max(mss) if args.exchange else sum(mss)
    # Responsiveness model (context for the paper's E6): the
    # schedule is fixed by the virtual clock (R17); each swap's MEASURED
    # device time is put on the critical path of the iteration that issued it
    # (no overlap: "GPUs are idle while they wait for the paged data",
    # P:305-308), and delays are absorbed by idle gaps:
    #   E_start(i) = max(V_start(i), E_end(i-1)) + swaps(i);  E_end(i) = E_start(i) + cost(i)
    e_end, prev = [], 0.0
    for i, tok in enumerate(it_tokens):
        e0 = max(v_start[i], prev) + swap_ms_at[i] / 1e3
        prev = e0 + 0.020 + 40e-6 * tok
        e_end.append(prev)
    bytes_out, bytes_in = st["blocks_out"] * U, st["blocks_in"] * U
    # NEXT-1 moves (reclaim lender -> host, re-offer host -> lender): device time per call
    mig = [(k, n, ctx.ticket_elapsed(tk)) for k, n, tk, _ in st["swap_calls"] if k in ("reclaim", "migrate") and n]

    def pct(xs, q):
        xs = sorted(xs)
        return round(xs[min(len(xs) - 1, int(q * len(xs)))], 4) if xs else None

    ttft = [e_end[first_it[p]] - arrival[p] for p in first_it]
    tpot = [(e_end[last_it[p]] - e_end[first_it[p]]) / (plen[p][1] - 1) for p in last_it
            if p in first_it and plen[p][1] > 1]
    res = {
        "config": f"configs[2] bursty trace (seed {args.trace_seed}, {len(trace)} requests, 25 @ 2.5/s then 5/s for 60 s "
                  "then 2.5/s for 15 s), Llama-3-8B KV shape, NB=4152 (8.1 GiB), b=512, k=8",
        "policy": args.policy,
        "mode": args.policy if args.policy != "cfs-peer" else
        ("self-lender (1 GPU)" if ws == 1 else ("IPC lender process, same GPU" if shared else "IPC peer lender GPU 1")),
        "iterations": st["iters"], "virtual_s": round(st["vclock"], 3), "wall_s": round(wall, 3),
        "swap_out_calls": sum(1 for x in swap_events if x[0] == "out"),
        "swap_in_calls": sum(1 for x in swap_events if x[0] == "in"),
        "bytes_out": bytes_out, "bytes_in": bytes_in,
        "swap_device_ms": {k: round(v, 3) for k, v in dev_ms.items()},
        "swap_GBps": {k: round((bytes_out if k == "out" else bytes_in) / max(v, 1e-9) / 1e6, 1)
                      for k, v in dev_ms.items() if v > 0},
        "kernel_launches": launches,
        "streams": ("serial (one stream)" if args.serial else "decode + swap streams (tickets)")
                   + (" + exchange (preempt/resume on two streams)" if args.exchange else ""),
        "proxy_gb_per_iteration": args.proxy_gb,
        "verify_mismatches": int(mism.item()),
        "responsiveness_model_s": {"ttft_p50": pct(ttft, 0.5), "ttft_p99": pct(ttft, 0.99),
                                   "ttft_max": pct(ttft, 1.0), "tpot_p50": pct(tpot, 0.5),
                                   "tpot_p99": pct(tpot, 0.99), "makespan": round(e_end[-1], 3) if e_end else None,
                                   "swap_on_critical_path_s": round(sum(swap_ms_at) / 1e3, 3)},
    }
    if elastic:
        res["elastic"] = {"t_reclaim": elastic["t_reclaim"], "t_relend": elastic["t_relend"],
                          "moves": [{"kind": k, "blocks": n, "ms": round(ms, 3),
                                     "GBps": round(n * U / ms / 1e6, 1)} for k, n, ms in mig]}
    outs = [ms / np_ for k, ms, n, np_ in per_block_ms if k == "out"]
    ins = [ms / np_ for k, ms, n, np_ in per_block_ms if k == "in"]
    if outs and ins:
        so, si = sorted(outs), sorted(ins)
        res["per_prompt_ms"] = {"preempt_p50": round(statistics.median(so), 4),
                                "preempt_p99": round(so[min(len(so) - 1, int(0.99 * len(so)))], 4),
                                "resume_p50": round(statistics.median(si), 4),
                                "resume_p99": round(si[min(len(si) - 1, int(0.99 * len(si)))], 4)}
    if args.check_oracle:
        from oracle import sim as osim
        o = osim.run(trace, osim.SimConfig(NB=NB, lender_slots=lend_bytes // U if args.policy == "cfs-peer" else 0,
                                           host_slots=(args.host_gib << 30) // U,
                                           policy="fcfs" if pol == POLICY_FCFS else "cfs",
                                           elastic=(elastic["t_reclaim"], elastic["t_relend"]) if elastic else None,
                                           relend_slots=(args.lender_gib << 30) // U))
        res["oracle_log_equal"] = (log == o.log)
        res["oracle_calls"] = len(o.log)
    print(json.dumps(res), flush=True)
    if ws == 2:
        import torch.distributed as dist
        ctx.close()
        if lend_dev == aqua.MAPPED:
            aqua.ipc_close(devi, lend_ptr)
        dist.barrier()
        dist.barrier()
        dist.destroy_process_group()
    if res["verify_mismatches"]:
        raise SystemExit("KV pattern mismatch after resume")


if __name__ == "__main__":
    main()
