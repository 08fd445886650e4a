"""Cross-process lending on one GPU (-m gpu): a lender process offers HBM
through a CUDA IPC handle, a borrower process maps it (aqua_ipc_import ->
aqua_lend(AQUA_MAPPED)) and pages a prompt into it with the fused kernel.
The LENDER then checks the image in its own memory against the oracle's
closed-form words -- the same code path the 2-GPU pairs use (with peer HBM
instead of the same HBM)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

L, bs, H, D, NB, NBLK, SEED = 2, 16, 2, 64, 64, 40, 4242


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, q, ldev=0):
    import torch
    import torch.distributed as dist
    from oracle import pattern as opat
    from paper_2407_21255_b200 import aqua
    from paper_2407_21255_b200.pairing import exchange
    from workloads import block_permutation

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(ldev if rank == 0 else 0)
    S = bs * H * D * 2
    U = 2 * L * S
    try:
        if rank == 0:                                   # lender (producer)
            ptr = aqua.ipc_alloc(ldev, NBLK * U)
            exchange((aqua.ipc_export(ptr), NBLK * U))
            dist.barrier()                              # borrower swaps out
            dist.barrier()
            torch.cuda.synchronize()

            class _Dev:   # view the lent allocation without copying through the library
                __cuda_array_interface__ = {"shape": (NBLK * U,), "typestr": "|u1", "data": (ptr, False),
                                            "version": 3}

            host = torch.as_tensor(_Dev(), device="cuda").cpu().numpy()
            img = host.reshape(NBLK, L, 2, bs, H, D * 2)
            bad = 0
            bt_len = NBLK
            for j in range(bt_len):
                for l in range(L):
                    for kv in (0, 1):
                        for i in range(bs):
                            w = opat.token_words(SEED, 7, j * bs + i, l, kv, H, D).reshape(-1).view(np.uint8)
                            bad += not np.array_equal(img[j, l, kv, i].reshape(-1), w)
            dist.barrier()                              # borrower closes its mapping
            aqua.ipc_free(ldev, ptr)
            q.put(("lender", bad))
        else:                                           # borrower (consumer)
            got = exchange(None)
            handle, nbytes = got[0]
            layers = [torch.zeros(2 * NB * S, dtype=torch.uint8, device="cuda") for _ in range(L)]
            ctx = aqua.Ctx(0, L, bs, H, D, 2, NB, [x.data_ptr() for x in layers])
            mapped = aqua.ipc_import(0, handle)
            assert ctx.lend(aqua.MAPPED, mapped, nbytes) == NBLK
            info = ctx.arena_info(aqua.LOC_PEER)
            assert info["device"] == ldev and info["peer"] == (ldev != 0)
            assert info["probe"] == (7 if ldev != 0 else -1)
            ctx.adopt_blocks(7, block_permutation(NB, NBLK, seed=3).tolist())
            ctx.kv_fill_pattern(7, 0, NBLK * bs, SEED)
            tk = ctx.swap_out([7])
            ctx.sync(tk)
            assert ctx.query(7)[1] == aqua.LOC_PEER
            dist.barrier()
            dist.barrier()                              # lender has checked its memory
            for x in layers:
                x.fill_(0x5A)
            new, tk = ctx.swap_in([7])
            cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
            ctx.kv_verify_pattern(7, NBLK * bs, SEED, cnt.data_ptr())
            torch.cuda.synchronize()
            ctx.close()
            aqua.ipc_close(0, mapped)
            dist.barrier()
            q.put(("borrower", int(cnt.item())))
    except Exception as ex:  # report instead of hanging the other rank
        q.put(("error", repr(ex)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ldev", [0, 1])
def test_ipc_lend_across_processes(ldev):
    """ldev = 1: the lender process offers HBM of GPU 1 and the borrower on
    GPU 0 maps it -- the NVLink path of the 2-8 GPU bench (skipped on a
    one-GPU box)."""
    import torch
    if ldev >= torch.cuda.device_count():
        pytest.skip("needs 2 GPUs (peer lender over NVLink)")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, port, q, ldev)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert "error" not in out, out
    assert out["lender"] == 0, "lender arena does not hold the borrower's image"
    assert out["borrower"] == 0, "resume from lent memory corrupted the KV"


@pytest.mark.parametrize("roles", ["both", "split"])
def test_bench_two_ranks_sharing_one_gpu(roles):
    """bench.py's N > 1 path end to end (the one the driver's scaling run
    takes on 2-8 GPUs): torchrun with 2 ranks, pairing, IPC-lending and
    paging the 32K-token prompt into the partner's memory; on one GPU
    (AQUA_BENCH_SHARED_GPU=1) the ranks share it.  roles "both": each rank
    borrows from the other; "split": rank 0 borrows, rank 1 only lends
    (configs[3]'s roles).  The line must carry the north_star block (per
    pair per direction, fractions of 900 and 770), per-rank latencies and a
    clean pattern verify."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, AQUA_BENCH_SHARED_GPU="1", MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(root, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-host-baselines", "--no-cpu-baseline",
           "--roles", roles]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["pairing"] == [1, 0]
    assert [p["rank"] for p in line["per_rank"]] == [0, 1]
    assert line["parity"].startswith("pattern verify: 0 mismatching words")
    assert line["roofline"]["bound"] == "nvlink" and line["roofline"]["peak"] == 770.0
    assert line["roofline"]["nominal_peak"] == 900.0
    ns = line["north_star"]
    assert ns["roles"] == roles and ns["pairs"] == (2 if roles == "both" else 1)
    assert ns["frac_of_900"]["swap_out"] > 0 and ns["frac_of_770_measured"]["swap_in"] > 0
    pr0 = line["per_rank"][0]
    assert pr0["preempt_resume_device_ms"] > 0 and pr0["preempt_resume_host_p50_ms"] > 0
    if roles == "split":
        assert line["per_rank"][1]["mode"] == "lender for rank0" and "swap_out_GBps" not in line["per_rank"][1]
    else:
        assert line["per_rank"][1]["swap_out_GBps"] > 0
