"""N>1 host logic on CPU with gloo, world_size 2: pairing and the
setup-time exchange of IPC handles (the data path itself needs GPUs)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2407_21255_b200.pairing import partner


def test_partner_matching():
    assert [partner(r, 8) for r in range(8)] == [1, 0, 3, 2, 5, 4, 7, 6]
    assert [partner(r, 3) for r in range(3)] == [1, 0, 2]
    assert partner(0, 1) == 0
    no = [[True, False], [False, True]]
    assert partner(0, 2, no) == 0
    # a perfect matching: partner(partner(r)) == r
    for w in range(1, 9):
        assert all(partner(partner(r, w), w) == r for r in range(w))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2407_21255_b200.pairing import exchange, partner
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    handle = bytes([rank]) * 64                       # stands in for cudaIpcMemHandle_t
    got = exchange((rank, handle, 1 << 30))
    p = partner(rank, world)
    q.put((rank, p, got[p]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_handle_exchange_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == 1 and res[0][2] == (1, bytes([1]) * 64, 1 << 30)
    assert res[1][1] == 0 and res[1][2] == (0, bytes([0]) * 64, 1 << 30)


def test_best_matching_from_measured_matrix():
    from paper_2407_21255_b200.pairing import best_matching
    n = 8
    uniform = [[0 if i == j else 770.0 for j in range(n)] for i in range(n)]
    assert best_matching(uniform) == [1, 0, 3, 2, 5, 4, 7, 6]        # NVSwitch: lowest-index matching
    # a slow link between 0 and 1 (and 2-3) steers the matching elsewhere
    bw = [row[:] for row in uniform]
    bw[0][1] = bw[1][0] = 100.0
    bw[2][3] = bw[3][2] = 100.0
    m = best_matching(bw)
    assert all(m[m[i]] == i for i in range(n)) and m[0] != 1 and m[2] != 3
    assert min(bw[i][m[i]] for i in range(n)) == 770.0
    # unreachable pairs are never chosen; odd counts self-lend one GPU
    bw3 = [[0, 0, 500.0], [0, 0, 0], [500.0, 0, 0]]
    assert best_matching(bw3) == [2, 1, 0]


def _all_matchings(n):
    """Every perfect matching of range(n) (odd n: one self-paired), as partner lists."""
    def rec(free, part):
        if not free:
            yield list(part)
            return
        i, rest = free[0], free[1:]
        if len(free) % 2 == 1:
            part[i] = i
            yield from rec(rest, part)
        for k, j in enumerate(rest):
            part[i], part[j] = j, i
            yield from rec(rest[:k] + rest[k + 1:], part)
        part[i] = -1
    yield from rec(list(range(n)), [-1] * n)


def test_pairing_objective_is_max_min_of_both_directions():
    """the pairing maximises the slowest pair's link, a pair's
    link being the slower of its two directions.  Brute force over every
    matching / assignment on random ASYMMETRIC matrices; and a case where
    maximising the total would pick a different matching."""
    import itertools
    import random
    from paper_2407_21255_b200.pairing import best_bipartite, best_matching

    def link(bw, i, j):
        return min(bw[i][j], bw[j][i])

    # the total (sum) would prefer {0-1, 2-3}: 2 x 200 + 2 x 10 = 420 > 400
    bw = [[0, 200, 100, 0], [200, 0, 0, 100], [100, 0, 0, 10], [0, 100, 10, 0]]
    assert best_matching(bw) == [2, 3, 0, 1]
    for seed in range(20):
        rnd = random.Random(seed)
        n = rnd.choice([4, 5, 6])
        bw = [[0 if i == j else rnd.choice([50.0, 300.0, 500.0, 770.0]) for j in range(n)] for i in range(n)]
        m = best_matching(bw)
        got = min((link(bw, i, m[i]) for i in range(n) if m[i] != i), default=float("inf"))
        want = max(min((link(bw, i, q[i]) for i in range(n) if q[i] != i), default=float("inf"))
                   for q in _all_matchings(n))
        assert got == want, (seed, bw, m)
        if n % 2 == 0:
            half = n // 2
            mb = best_bipartite(bw, list(range(half)), list(range(half, n)))
            got = min(link(bw, b, mb[b]) for b in range(half))
            want = max(min(link(bw, b, l) for b, l in zip(range(half), p))
                       for p in itertools.permutations(range(half, n)))
            assert got == want, (seed, bw, mb)


def test_best_bipartite_split_roles():
    """configs[3]'s roles: borrowers 0-3 each page to one of lenders 4-7."""
    import itertools
    from paper_2407_21255_b200.pairing import best_bipartite
    n = 8
    uniform = [[0 if i == j else 770.0 for j in range(n)] for i in range(n)]
    assert best_bipartite(uniform, [0, 1, 2, 3], [4, 5, 6, 7]) == [4, 5, 6, 7, 0, 1, 2, 3]
    bw = [row[:] for row in uniform]
    bw[0][4] = bw[4][0] = 90.0                       # a slow link is avoided
    m = best_bipartite(bw, [0, 1, 2, 3], [4, 5, 6, 7])
    assert m[0] != 4 and all(m[m[i]] == i for i in range(n)) and sorted(m[:4]) == [4, 5, 6, 7]
    # brute-force check of the max-min objective on a random matrix
    import random
    rnd = random.Random(3)
    bw = [[0 if i == j else rnd.choice([300.0, 500.0, 770.0]) for j in range(n)] for i in range(n)]
    m = best_bipartite(bw, [0, 1, 2, 3], [4, 5, 6, 7])
    got = min(min(bw[b][m[b]], bw[m[b]][b]) for b in range(4))
    want = max(min(min(bw[b][l], bw[l][b]) for b, l in zip(range(4), p))
               for p in itertools.permutations(range(4, 8)))
    assert got == want
    with pytest.raises(ValueError):
        best_bipartite(uniform, [0, 1], [2])


def _tp_worker(rank, world, port, q):
    """Two TP ranks in dry-run mode with their own KV-head shard: the
    replicated native scheduler gives both the same call log."""
    import hashlib
    import torch.distributed as dist
    from paper_2407_21255_b200 import aqua
    from paper_2407_21255_b200.cfs import Scheduler
    from paper_2407_21255_b200.driver import run_trace
    from workloads import burst_trace
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    FAKE = 1 << 40
    H = 8 // world
    c = aqua.Ctx(aqua.DRYRUN, 4, 16, H, 128, 2, 120, [FAKE + l * (1 << 34) for l in range(4)])
    c.lend(0, FAKE * 8, 3000 * c.U)
    tr = burst_trace(seed=3, burst_s=6.0, tail_s=2.0, prompt=(300, 0.8, 1, 900), output=(40, 0.7, 1, 200))
    log, _ = run_trace(tr, c, Scheduler(NB=120, bs=16))
    hs = [None] * world
    dist.all_gather_object(hs, hashlib.sha256(repr(log).encode()).hexdigest())
    q.put((rank, hs, sum(1 for e in log if e[0] == "swap_out")))
    dist.destroy_process_group()


def test_tp_ranks_replicated_schedule():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_tp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=180) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, hs, nout in res:
        assert len(set(hs)) == 1 and nout > 0


def test_reference_arm_under_torchrun_world2():
    """bench.py --impl reference under torchrun (N=2, CPU only): rank 0 alone
    times the oracle and prints ONE line; the other rank exits 0 without work."""
    import json
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(root, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["value"] > 0
    assert lines[0]["n_gpus"] == 2 and lines[0]["cpu_baseline"]["kind"] == "oracle"
