"""GPU parity (-m gpu): libaqua's sm_100a kernels against the CPU oracle,
byte for byte (tolerance 0), through the C ABI.

Whole-buffer comparison (pool, GPU lender arena, host arena) after every
call for C1 (BASELINE configs[0]) and randomised op sequences at sizes that
span several TMA stages and a ragged tail; the full-size C2 configuration is
checked on sampled chunks against the oracle's closed-form pattern words and
by the any-size restore property (pattern verify kernel)."""
import json
import os
import random

import numpy as np
import pytest
import torch

from oracle import kvpool as kp
from oracle import pattern as opat
from paper_2407_21255_b200 import aqua
from workloads import block_permutation

from gpu_util import Rig

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
ENGINES = {"tma": aqua.KERNEL_TMA, "ldst": aqua.KERNEL_LDST, "per_chunk": aqua.BASE_PER_CHUNK,
           "gather_temp": aqua.BASE_GATHER_TEMP, "ce_host": aqua.KERNEL_CE_HOST,
           "tma_dyn": aqua.KERNEL_TMA, "tma_dyn1": aqua.KERNEL_TMA, "tma_static": aqua.KERNEL_TMA,
           "tma_hybrid": aqua.KERNEL_TMA, "ldst_small": aqua.KERNEL_LDST, "auto": aqua.KERNEL_AUTO}
# the engines and schedules the library can run (round 1's AUTO-unused experiments were retired in round 2)
KERNEL_ENGINES = ["auto", "tma", "tma_dyn", "tma_dyn1", "tma_static", "tma_hybrid", "ldst", "ldst_small"]


def _engine(ctx, name):
    """Select an engine; "auto" the library's AUTO policy (engine and schedule), "tma" the AUTO schedule of the
    TMA ring, "tma_dyn" / "tma_dyn1" its claimed batches
    of 8 / 1 ring units, "tma_static" one contiguous item range per CTA, "tma_hybrid" the ring plus 8 LDST
    warps claiming batches of the same launch, "ldst_small" the small-chunk register kernel (rounds of whole
    chunks of 512 B .. 4 KiB; other sizes fall back to the pipelined LDST kernel)."""
    ctx.set_option(aqua.OPT_KERNEL, ENGINES[name])
    ctx.set_option(aqua.OPT_TMA_VARIANT, 3 if name == "tma_hybrid" else 0)
    ctx.set_option(aqua.OPT_LDST_VARIANT, 3 if name == "ldst_small" else 2)
    if name in ("tma_dyn", "tma_dyn1", "tma_static"):
        ctx.set_option(aqua.OPT_TMA_SCHED, {"tma_dyn": 8, "tma_dyn1": 1, "tma_static": 0}[name])


def _ops(rig, ops, stream=0):
    """Apply ops to both sides and compare everything after each."""
    c, o = rig.ctx, rig.opool
    for name, arg in ops:
        if name == "alloc":
            assert c.alloc_blocks(*arg, stream=stream) == o.alloc_blocks(*arg)
        elif name == "adopt":
            c.adopt_blocks(*arg, stream=stream)
            o.adopt_blocks(*arg)
        elif name == "out":
            c.swap_out(arg, stream)
            res = o.swap_out(arg)
            for pid, loc, slots in res:
                assert c.query(pid, with_ids=True)[1:] == (loc, len(slots), slots)
        elif name == "in":
            new, _ = c.swap_in(arg, stream)
            assert new == o.swap_in(arg)
        elif name == "free":
            c.free(arg, stream)
            o.free_prompt(arg)
        rig.assert_bytes_equal(f"after {name} {arg}")


@pytest.mark.parametrize("engine", list(ENGINES))
@pytest.mark.parametrize("variant", ["lender12", "lender8"])
def test_c1_bytes(engine, variant):
    g = json.load(open(os.path.join(GOLD, "c1_script.json")))
    v = g[variant]
    rig = Rig(**g["layout"], lender_slots=v["lender_slots"], host_slots=v.get("host_slots", 0))
    _engine(rig.ctx, engine)
    s = torch.cuda.Stream()
    ops = [("alloc", (p, 4)) for p in range(8)]
    ops += [("out", g["swap_out"]), ("alloc", (100, 6)), ("in", g["swap_in"]), ("free", 100)]
    _ops(rig, ops, stream=s.cuda_stream if engine != "tma" else 0)
    for pid, ids in g["expected_swap_in_ids"].items():
        assert rig.ctx.query(int(pid), with_ids=True)[3] == ids


SHAPES = {
    # (L, bs, H, D): S bytes -> TMA pieces at the default 16 KiB piece
    "tiny_256B": (1, 16, 1, 8),          # S = 256 B (one small piece)
    "ragged_10KiB": (3, 16, 5, 64),      # S = 10 KiB: TMA pieces 4K, 4K, 2K (piece option 4096)
    "llama_bs32": (4, 32, 8, 128),       # S = 64 KiB (4 pieces)
    "odd_48KiB": (2, 16, 12, 128),       # S = 48 KiB (3 pieces)
    "c4_shape": (5, 16, 2, 128),         # S = 8 KiB (Llama-70B TP4 chunk): TMA units of 4,4,2 chunks
    "l3_8KiB": (3, 16, 2, 128),          # S = 8 KiB, 6 chunks per block: units of 4,2
    "fp8_kv": (2, 16, 8, 128, 1),        # e = 1 (FP8 KV cache): S = 16 KiB
    "fp32_kv": (2, 16, 4, 128, 4),       # e = 4: S = 32 KiB (one full stage)
    "bs128": (1, 128, 8, 128),           # S = 256 KiB: 8 pieces per chunk
    "s1k": (3, 16, 1, 32),               # S = 1 KiB: 4 chunks per register round (hybrid packing)
    "s2k": (2, 16, 1, 64),               # S = 2 KiB: 2 chunks per register round
    "s512": (5, 16, 1, 16),              # S = 512 B: 8 chunks per register round, ragged descriptor crossings
}


# AQUA_FUZZ_SEEDS / AQUA_FUZZ_OPS widen the random sequences for one-off long fuzz runs
# (scripts/gpu_runs/r02_run41.sh); the suite runs 2 seeds x 25 ops.
FUZZ_SEEDS = list(range(int(os.environ.get("AQUA_FUZZ_SEEDS", "2"))))
FUZZ_OPS = int(os.environ.get("AQUA_FUZZ_OPS", "25"))


@pytest.mark.parametrize("shape", list(SHAPES))
@pytest.mark.parametrize("engine", KERNEL_ENGINES)
@pytest.mark.parametrize("seed", FUZZ_SEEDS)
@pytest.mark.parametrize("ctas", [0, 3])
def test_random_sequences_bytes(shape, engine, seed, ctas):
    """ctas=3 forces many units per CTA (TMA: grouped chunks split at ragged
    descriptor and CTA-range boundaries)."""
    L, bs, H, D, *e = SHAPES[shape]
    rnd = random.Random(seed * 31 + len(shape))
    NB = 24
    rig = Rig(L=L, bs=bs, H=H, D=D, e=(e or [2])[0], NB=NB, lender_slots=10, host_slots=8, seed=seed)
    _engine(rig.ctx, engine)
    rig.ctx.set_option(aqua.OPT_MAX_CTAS, ctas)
    if engine.startswith("tma") and shape == "ragged_10KiB":
        rig.ctx.set_option(aqua.OPT_TMA_PIECE, 4096)     # S = 10 KiB -> pieces 4K, 4K, 2K
    pids = list(range(5))
    ops = []
    state = {}
    for _ in range(FUZZ_OPS):
        k = rnd.random()
        p = rnd.choice(pids)
        if k < 0.35:
            ops.append(("alloc", (p, rnd.randint(0, 4))))
        elif k < 0.6:
            ops.append(("out", rnd.sample(pids, rnd.randint(1, 3))))
        elif k < 0.85:
            ops.append(("in", rnd.sample(pids, rnd.randint(1, 3))))
        else:
            ops.append(("free", p))
    c, o = rig.ctx, rig.opool
    for op in ops:
        try:
            _ops(rig, [op])
        except (kp.AquaError, aqua.AquaError) as e:
            # errors must agree and change nothing on either side
            code_o = code_c = None
            name, arg = op
            try:
                {"alloc": lambda: o.alloc_blocks(*arg), "out": lambda: o.swap_out(arg),
                 "in": lambda: o.swap_in(arg), "free": lambda: o.free_prompt(arg)}[name]()
            except kp.AquaError as eo:
                code_o = eo.code
            try:
                {"alloc": lambda: c.alloc_blocks(*arg), "out": lambda: c.swap_out(arg),
                 "in": lambda: c.swap_in(arg, cap=4096), "free": lambda: c.free(arg)}[name]()
            except aqua.AquaError as ec:
                code_c = ec.code
            assert code_o is not None and code_o == code_c == e.code, (op, code_o, code_c)
            rig.assert_bytes_equal(f"after failed {op}")


@pytest.mark.parametrize("engine", ["auto", "tma", "tma_dyn1", "tma_hybrid", "ldst", "ldst_small", "ce_host"])
@pytest.mark.parametrize("D", [64, 8, 16])
def test_block_major_layout_bytes(engine, D):
    """Block-major layout ([NB][2][bs][H][D] per layer, kv_plane_stride = S):
    a layer's K and V chunks are adjacent in pool and image and move as one
    2S chunk (S = 4 KiB, and 256 / 512 B where the register movers pack
    several merged chunks per round)."""
    L, bs, H, NB = 3, 16, 2, 12
    S = bs * H * D * 2
    rig = Rig(L=L, bs=bs, H=H, D=D, NB=NB, lender_slots=6, host_slots=6, kv_plane_stride=S, block_stride=2 * S)
    _engine(rig.ctx, engine)
    _ops(rig, [("adopt", (1, [5, 0, 3])), ("alloc", (2, 4)), ("out", [1, 2]), ("alloc", (3, 2)), ("in", [2, 1])])


def test_block_major_layerwise_bytes():
    """Layer-wise swaps (chunk ranges of whole layers) on the merged K+V layout."""
    L, bs, H, D, NB = 5, 16, 1, 32, 20
    S = bs * H * D * 2
    rig = Rig(L=L, bs=bs, H=H, D=D, NB=NB, lender_slots=8, host_slots=0, kv_plane_stride=S, block_stride=2 * S)
    c, o = rig.ctx, rig.opool
    perm = block_permutation(NB, 7, seed=4).tolist()
    c.adopt_blocks(3, perm)
    o.adopt_blocks(3, perm)
    c.swap_out_layers([3], 2)
    o.swap_out([3])
    rig.assert_bytes_equal("layered swap_out, block-major")
    new, _ = c.swap_in_layers([3], 2)
    assert new == o.swap_in([3])
    rig.assert_bytes_equal("layered swap_in, block-major")


def test_adversarial_reuse_on_other_streams():
    """R7: freed blocks / slots are handed out again at once and overwritten
    on another stream while the swap that read them may still be in flight;
    the library's stream waits keep the result equal to sequential
    execution."""
    L, bs, H, D, NB = 4, 16, 8, 128, 64          # S = 32 KiB, U = 256 KiB
    rig = Rig(L=L, bs=bs, H=H, D=D, NB=NB, lender_slots=32, host_slots=0)
    c, o = rig.ctx, rig.opool
    s_swap, s_dec = torch.cuda.Stream(), torch.cuda.Stream()
    for p in range(4):
        assert c.alloc_blocks(p, 16, s_dec.cuda_stream) == o.alloc_blocks(p, 16)
    torch.cuda.synchronize()
    for rnd in range(6):
        # big swap out on s_swap ...
        s_swap.wait_stream(s_dec)
        c.swap_out([0, 1], s_swap.cuda_stream)
        o.swap_out([0, 1])
        # ... its blocks are immediately reallocated and scribbled on s_dec
        ids = c.alloc_blocks(10 + rnd, 32, s_dec.cuda_stream)
        assert ids == o.alloc_blocks(10 + rnd, 32)
        with torch.cuda.stream(s_dec):
            val = (rnd * 37 + 11) % 256
            for b in ids:
                for l in range(L):
                    for kv in (0, 1):
                        off = kv * rig.lay.P_kv + b * rig.lay.P_b
                        rig.layers[l][off:off + rig.lay.S].fill_(val)
                        o.chunk(l, kv, b)[:] = val
        c.free(10 + rnd, s_dec.cuda_stream)
        o.free_prompt(10 + rnd)
        # swap back in on the swap stream (must wait for the scribbles that
        # last touched the reused blocks), then its slots are reused by a
        # swap_out on the decode stream
        new, t = c.swap_in([1, 0], s_swap.cuda_stream)
        assert new == o.swap_in([1, 0])
        c.swap_out([2], s_dec.cuda_stream)
        o.swap_out([2])
        new, t2 = c.swap_in([2], s_swap.cuda_stream)
        assert new == o.swap_in([2])
    rig.assert_bytes_equal("adversarial")


@pytest.mark.parametrize("late", ["swap_out", "scribble", "swap_in", "slot_reuse"])
def test_adversarial_reuse_with_a_delayed_stream(late):
    """R7 made deterministic: a ~20 ms sleep kernel queued on one stream makes
    the operation that was ENQUEUED first run LAST unless the library orders
    the later one after it.  Each case delays one step of a reuse chain:
      swap_out   -- a swap_out reads blocks that alloc_blocks hands out again
                    at once and the caller overwrites on another stream (A4);
      scribble   -- the caller's writes to reused blocks are late; the
                    swap_in that receives those blocks after aqua_free must
                    wait for them (free records the caller's stream);
      swap_in    -- a swap_in reads lender slots that a swap_out on another
                    stream reuses right after (A7);
      slot_reuse -- the swap_out into the reused slots is late relative to
                    nothing (control: must still equal sequential execution).
    Without the library's waits each case would read or overwrite the wrong
    bytes; the result must equal the oracle's sequential run."""
    L, bs, H, D, NB = 4, 16, 8, 128, 64          # S = 32 KiB, U = 256 KiB
    rig = Rig(L=L, bs=bs, H=H, D=D, NB=NB, lender_slots=32, host_slots=0)
    c, o = rig.ctx, rig.opool
    s_swap, s_dec = torch.cuda.Stream(), torch.cuda.Stream()
    delay = 40_000_000                            # ~20 ms at 1.9 GHz: longer than the host's enqueueing
    for p in range(4):
        assert c.alloc_blocks(p, 16, s_dec.cuda_stream) == o.alloc_blocks(p, 16)
    torch.cuda.synchronize()
    for rnd in range(3):
        s_swap.wait_stream(s_dec)
        if late == "swap_out":
            with torch.cuda.stream(s_swap):
                torch.cuda._sleep(delay)
        c.swap_out([0, 1], s_swap.cuda_stream)
        o.swap_out([0, 1])
        ids = c.alloc_blocks(10 + rnd, 32, s_dec.cuda_stream)
        assert ids == o.alloc_blocks(10 + rnd, 32)
        with torch.cuda.stream(s_dec):
            if late == "scribble":
                torch.cuda._sleep(delay)
            val = (rnd * 37 + 11) % 256
            for l in range(L):
                for kv in (0, 1):
                    for b in ids:
                        off = kv * rig.lay.P_kv + b * rig.lay.P_b
                        rig.layers[l][off:off + rig.lay.S].fill_(val)
                        o.chunk(l, kv, b)[:] = val
        c.free(10 + rnd, s_dec.cuda_stream)
        o.free_prompt(10 + rnd)
        if late == "swap_in":
            with torch.cuda.stream(s_swap):
                torch.cuda._sleep(delay)
        new, _ = c.swap_in([1, 0], s_swap.cuda_stream)
        assert new == o.swap_in([1, 0])
        if late == "slot_reuse":
            with torch.cuda.stream(s_dec):
                torch.cuda._sleep(delay)
        c.swap_out([2], s_dec.cuda_stream)
        o.swap_out([2])
        new, _ = c.swap_in([2], s_swap.cuda_stream)
        assert new == o.swap_in([2])
    rig.assert_bytes_equal(f"adversarial, late {late}")


def test_c2_full_size_sampled_and_restore():
    """BASELINE configs[1] in the bench's launch configuration: one 32K-token
    Llama-3-8B prompt (2048 blocks of U = 2 MiB) on a fragmented block table
    (seeded permutation of 4096), self-lender arena 4 GiB; plus the host arena
    for a second prompt.  Sampled chunks are compared with the oracle's
    closed-form words; the whole prompt with the pattern verify kernel."""
    L, bs, H, D, NB = 32, 16, 8, 128, 4096
    S = bs * H * D * 2
    lay = kp.Layout(L=L, bs=bs, H=H, D=D, e=2, NB=NB)
    dev = torch.device("cuda", 0)
    layers = [torch.zeros(lay.layer_bytes, dtype=torch.uint8, device=dev) for _ in range(L)]
    arena = torch.zeros(2048 * lay.U, dtype=torch.uint8, device=dev)
    c = aqua.Ctx(0, L, bs, H, D, 2, NB, [t.data_ptr() for t in layers])
    c.lend(0, arena.data_ptr(), 2048 * lay.U)
    c.lend(aqua.HOST, 0, 64 * lay.U)                      # library-owned pinned arena
    bt = block_permutation(NB, 2048, seed=2).tolist()
    c.adopt_blocks(7, bt)
    ntok, seed = 32768, 1234
    c.kv_fill_pattern(7, 0, ntok, seed)
    c.alloc_blocks(8, 64)
    c.kv_fill_pattern(8, 0, 64 * bs, seed)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    c.swap_out([7, 8])
    assert c.query(7)[1] == aqua.LOC_PEER and c.query(8)[1] == aqua.LOC_HOST
    slots = c.query(7, with_ids=True)[3]
    assert slots == list(range(2048))
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    img = arena.view(2048, L, 2, bs, H, D * 2)
    for _ in range(24):   # sampled chunks vs the oracle's words, token by token
        j = int(rng.integers(0, 2048))
        l = int(rng.integers(0, L))
        kv = int(rng.integers(0, 2))
        i = int(rng.integers(0, bs))
        t = j * bs + i
        want = opat.token_words(seed, 7, t, l, kv, H, D).reshape(-1).view(np.uint8).reshape(H, D * 2)
        assert np.array_equal(img[slots[j], l, kv, i].cpu().numpy(), want)
    # scribble over the freed pool, then resume into fresh blocks
    for t_ in layers:
        t_.fill_(0xA5)
    new, tk = c.swap_in([8, 7])
    assert new[0] == list(range(64)) and new[1] == list(range(64, 2112))
    c.kv_verify_pattern(7, ntok, seed, cnt.data_ptr())
    c.kv_verify_pattern(8, 64 * bs, seed, cnt.data_ptr())
    torch.cuda.synchronize()
    assert int(cnt.item()) == 0
    # a wrong seed is detected (the verifier is live)
    c.kv_verify_pattern(7, 16, seed + 1, cnt.data_ptr())
    torch.cuda.synchronize()
    assert int(cnt.item()) > 0


@pytest.mark.parametrize("cap", [0, 32])
def test_c4_full_size_sampled_and_restore(cap):
    """BASELINE configs[3] per TP rank (Llama-3-70B KV over TP4: L=80, 2 KV
    heads, S = 8 KiB) as bench.py --config c4 runs it: 32 prompts x 2048
    tokens swapped out and back in one call each (4,096 descriptors: staged
    upload, claimed batches of grouped chunks).  cap=32 caps the preemption
    at 32 SMs, where AUTO runs the hybrid ring + LDST warps.  Sampled chunks vs
    the oracle's closed-form words; every prompt restored (verify kernel)."""
    L, bs, H, D, NB = 80, 16, 2, 128, 8192
    lay = kp.Layout(L=L, bs=bs, H=H, D=D, e=2, NB=NB)
    dev = torch.device("cuda", 0)
    layers = [torch.zeros(lay.layer_bytes, dtype=torch.uint8, device=dev) for _ in range(L)]
    nblk = 4096
    arena = torch.zeros(nblk * lay.U, dtype=torch.uint8, device=dev)
    c = aqua.Ctx(0, L, bs, H, D, 2, NB, [t.data_ptr() for t in layers])
    c.lend(0, arena.data_ptr(), nblk * lay.U)
    perm = block_permutation(NB, NB, seed=2).tolist()
    c.adopt_blocks(1, perm[nblk:])                        # filler keeps the tables scattered
    pids = list(range(100, 132))
    seed = 77
    for i, pid in enumerate(pids):
        c.adopt_blocks(pid, perm[i * 128:(i + 1) * 128])
        c.kv_fill_pattern(pid, 0, 128 * bs, seed)
    c.set_option(aqua.OPT_MAX_CTAS, cap)
    c.swap_out(pids)
    c.set_option(aqua.OPT_MAX_CTAS, 0)
    torch.cuda.synchronize()
    rng = np.random.default_rng(1)
    img = arena.view(nblk, L, 2, bs, H, D * 2)
    for _ in range(24):
        pid = pids[int(rng.integers(0, 32))]
        slots = c.query(pid, with_ids=True)[3]
        jb = int(rng.integers(0, 128))
        l, kv, i = int(rng.integers(0, L)), int(rng.integers(0, 2)), int(rng.integers(0, bs))
        want = opat.token_words(seed, pid, jb * bs + i, l, kv, H, D).reshape(-1).view(np.uint8).reshape(H, D * 2)
        assert np.array_equal(img[slots[jb], l, kv, i].cpu().numpy(), want)
    for t_ in layers:
        t_.fill_(0x5A)
    c.free(1)
    new, _ = c.swap_in(pids[::-1])
    assert sorted(b for ids in new for b in ids) == list(range(nblk))
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    for pid in pids:
        c.kv_verify_pattern(pid, 128 * bs, seed, cnt.data_ptr())
    torch.cuda.synchronize()
    assert int(cnt.item()) == 0
    c.close()


def test_pattern_kernel_matches_oracle_words():
    rig = Rig(L=2, bs=16, H=2, D=64, NB=8, lender_slots=0)
    rig.ctx.adopt_blocks(3, [6, 2])
    rig.opool.adopt_blocks(3, [6, 2])
    rig.ctx.kv_fill_pattern(3, 5, 27, 99)
    opat.write_tokens(rig.opool, 3, 5, 27, 99)
    rig.assert_bytes_equal("pattern")


def test_errors_leave_state_unchanged_and_no_cpu_fallback():
    rig = Rig(L=2, bs=16, H=2, D=64, NB=8, lender_slots=2)
    c = rig.ctx
    c.alloc_blocks(1, 3)
    with pytest.raises(aqua.AquaError) as e:
        c.swap_out([1])                       # 3 blocks, lender has 2 slots, no host
    assert e.value.code == aqua.E_NOSPACE
    assert c.query(1)[0] == aqua.RESIDENT
    rig.opool.alloc_blocks(1, 3)
    rig.assert_bytes_equal("after NOSPACE")
    n0 = c.launch_count()
    c.alloc_blocks(2, 1)
    c.swap_out([2])
    assert c.launch_count() == n0 + 1         # the copy ran as one of our kernels


@pytest.mark.parametrize("engine", KERNEL_ENGINES)
@pytest.mark.parametrize("tier", ["small_inline", "big_inline", "staged_256", "staged_4064"])
def test_descriptor_tiers_bytes(engine, tier):
    """Descriptor passing, whole-buffer compare (both directions, fragmented
    table): calls of <= 256 blocks ride in the small parameter block, calls of
    <= AQUA_OPT_INLINE_MAX (default 4064) in the large-parameter launch, and
    larger calls go through the pinned staging ring (forced at 256 by the
    option, and at the default limit by a 4,200-block call)."""
    if tier == "staged_4064":
        NB, a, b, lend, host = 9000, 4100, 4300, 4400, 4400
    else:
        NB, a, b, lend, host = 700, 257 if tier != "small_inline" else 200, 600, 300, 400
    rig = Rig(L=2, bs=16, H=1, D=8, NB=NB, lender_slots=lend, host_slots=host)
    _engine(rig.ctx, engine)
    if tier == "staged_256":
        rig.ctx.set_option(aqua.OPT_INLINE_MAX, 256)
    assert rig.ctx.get_option(aqua.OPT_INLINE_MAX) == (256 if tier == "staged_256" else 4064)
    perm = block_permutation(NB, NB, seed=5).tolist()
    _ops(rig, [("adopt", (1, perm[:a])), ("adopt", (2, perm[a:b])), ("out", [1, 2]),
               ("alloc", (3, 50)), ("in", [2, 1]), ("out", [3, 1]), ("in", [1])])


def test_ticket_timing():
    rig = Rig(L=4, bs=16, H=8, D=128, NB=64, lender_slots=32)
    c = rig.ctx
    c.set_option(aqua.OPT_TIMING, 1)
    c.alloc_blocks(1, 32)
    t = c.swap_out([1])
    c.sync(t)
    ms = c.ticket_elapsed(t)
    assert 0.0 < ms < 100.0
    c.set_option(aqua.OPT_TIMING, 0)
    _, t2 = c.swap_in([1])
    c.sync(t2)
    with pytest.raises(aqua.AquaError) as e:
        c.ticket_elapsed(t2)
    assert e.value.code == aqua.E_STATE


@pytest.mark.parametrize("engine", KERNEL_ENGINES)
def test_migrate_reclaim_relend_bytes(engine):
    """NEXT-1 on the GPU: images move lender -> host (reclaim) and back
    (re-offer) -- AUTO on the copy engines, explicit engines through the fused
    arena->arena kernel -- byte for byte with the
    oracle; resumes from either place restore the blocks."""
    import torch
    from workloads import kv_random_bytes
    rig = Rig(L=3, bs=16, H=4, D=64, NB=40, lender_slots=12, host_slots=16)
    c, o = rig.ctx, rig.opool
    _engine(c, engine)
    _ops(rig, [("alloc", (1, 5)), ("alloc", (2, 3)), ("alloc", (3, 4)), ("out", [1, 3]), ("out", [2])])
    n0 = c.launch_count()
    t = c.migrate([3], aqua.LOC_HOST)
    o.migrate([3], kp.LOC_HOST)
    rig.assert_bytes_equal("migrate 3 -> host")
    # AUTO moves slot-contiguous images on the copy engines (no kernel); an explicit engine launches it
    assert (c.launch_count() - n0) == (0 if engine == "auto" else 1)
    t = c.reclaim()
    moved = o.reclaim()
    assert [p for p, _ in moved] == [1, 2]
    c.sync(t)
    assert c.counts()[1] == -1 and c.query(1)[1] == aqua.LOC_HOST
    torch.cuda.synchronize()
    assert np.array_equal(rig.host.numpy(), o.host.data)
    # re-offer a new lender and move two images back
    U = rig.lay.U
    g = kv_random_bytes(8 * U, seed=77)
    rig.peer = torch.from_numpy(g.copy()).cuda()
    o.lend(kp.LOC_PEER, 8 * U, g.copy())
    assert c.lend(0, rig.peer.data_ptr(), 8 * U) == 8
    c.migrate([2, 1], aqua.LOC_PEER)
    assert o.migrate([2, 1], kp.LOC_PEER) == [(2, [0, 1, 2]), (1, [3, 4, 5, 6, 7])]
    rig.assert_bytes_equal("migrate back")
    _ops(rig, [("in", [1, 2, 3]), ("out", [2])])


@pytest.mark.parametrize("engine", KERNEL_ENGINES)
def test_prefix_cache_bytes(engine):
    """NEXT-2 on the GPU: store a cached prefix (copy), load it into three
    new prompts, reclaim moves it to the host, load again -- whole buffers
    byte-equal to the oracle after every call."""
    rig = Rig(L=3, bs=16, H=4, D=64, NB=48, lender_slots=12, host_slots=12)
    c, o = rig.ctx, rig.opool
    _engine(c, engine)
    _ops(rig, [("adopt", (5, [40, 3, 17, 8, 22]))])
    c.prefix_store(9, 5, 4)
    assert o.prefix_store(9, 5, 4) == (kp.LOC_PEER, [0, 1, 2, 3])
    rig.assert_bytes_equal("prefix store")
    for dst in (100, 101, 102):
        ids, _ = c.prefix_load(9, dst)
        assert ids == o.prefix_load(9, dst)
        rig.assert_bytes_equal(f"prefix load {dst}")
    _ops(rig, [("out", [101])])
    c.reclaim()
    o.reclaim()
    assert c.prefix_query(9) == (aqua.LOC_HOST, o.prefixes[9].slots)
    ids, _ = c.prefix_load(9, 103)
    assert ids == o.prefix_load(9, 103)
    torch.cuda.synchronize()
    for l, t in enumerate(rig.layers):
        assert np.array_equal(t.cpu().numpy(), o.layers[l])
    assert np.array_equal(rig.host.numpy(), o.host.data)
    c.prefix_drop(9)
    o.prefix_drop(9)
    assert c.counts()[2] == len(o.host.free)


@pytest.mark.parametrize("layer_group", [1, 3, 4])
@pytest.mark.parametrize("nblk", [6, 300])
@pytest.mark.parametrize("where", ["lender", "host_ce"])
def test_layerwise_swaps_bytes(layer_group, nblk, where):
    """NEXT-3: swap_out/in split into per-layer-group launches give exactly the
    oracle's swap_out/swap_in bytes (inline and staged descriptors, ragged
    last group); each group has its own ticket, in issue order."""
    rig = Rig(L=4, bs=16, H=2, D=32, NB=2 * nblk + 8, lender_slots=nblk if where == "lender" else 0,
              host_slots=0 if where == "lender" else nblk)
    c, o = rig.ctx, rig.opool
    if where == "host_ce":
        c.set_option(aqua.OPT_KERNEL, aqua.KERNEL_CE_HOST)
    perm = block_permutation(2 * nblk + 8, nblk, seed=9).tolist()
    c.adopt_blocks(3, perm)
    o.adopt_blocks(3, perm)
    tks = c.swap_out_layers([3], layer_group)
    o.swap_out([3])
    assert len(tks) == -(-4 // layer_group) and tks == sorted(tks) and len(set(tks)) == len(tks)
    rig.assert_bytes_equal("layered swap_out")
    c.alloc_blocks(4, 5)
    o.alloc_blocks(4, 5)
    new, tks = c.swap_in_layers([3], layer_group)
    assert new == o.swap_in([3])
    c.sync(tks[0])
    assert c.ticket_done(tks[0])
    rig.assert_bytes_equal("layered swap_in")


def test_host_engines_switching_in_one_ctx():
    """The copy-engine host path's staging buffers survive engine switches in
    one ctx: CE_HOST, then the gather-temp baseline growing its own buffer,
    then AUTO (which picks CE_HOST for host-only calls), mixing whole-prompt
    and layer-wise calls whose per-descriptor range differs (S = 10 KiB, so
    the ranges do not divide the 256 MiB staging chunk).  Whole-buffer
    equality with the oracle after every call."""
    rig = Rig(L=3, bs=16, H=5, D=64, NB=96, lender_slots=0, host_slots=80, seed=4)
    c, o = rig.ctx, rig.opool
    rnd = random.Random(11)
    plan = ["ce", "ce_layers", "gather", "auto", "gather_big", "auto_layers", "ce", "auto", "auto_layers"]
    pids = list(range(6))
    for p in pids:
        n = rnd.randint(2, 9)
        assert c.alloc_blocks(p, n) == o.alloc_blocks(p, n)
    rig.assert_bytes_equal("setup")
    resident = set(pids)
    for step, mode in enumerate(plan):
        c.set_option(aqua.OPT_KERNEL, {"ce": aqua.KERNEL_CE_HOST, "ce_layers": aqua.KERNEL_CE_HOST,
                                       "gather": aqua.BASE_GATHER_TEMP, "gather_big": aqua.BASE_GATHER_TEMP,
                                       "auto": aqua.KERNEL_AUTO, "auto_layers": aqua.KERNEL_AUTO}[mode])
        k = len(pids) if mode == "gather_big" else rnd.randint(1, 3)
        outs = sorted(resident)[:k] if mode == "gather_big" else rnd.sample(sorted(resident), min(k, len(resident)))
        if outs:
            if mode.endswith("layers"):
                c.swap_out_layers(outs, 2)
            else:
                c.swap_out(outs)
            o.swap_out(outs)
            resident -= set(outs)
            rig.assert_bytes_equal(f"{mode} swap_out {outs}")
        ins = rnd.sample(sorted(set(pids) - resident), rnd.randint(1, len(set(pids) - resident)))
        if mode.endswith("layers"):
            new, _ = c.swap_in_layers(ins, 2)
        else:
            new, _ = c.swap_in(ins)
        assert new == o.swap_in(ins)
        resident |= set(ins)
        rig.assert_bytes_equal(f"{mode} swap_in {ins}")
    c.close()                       # explicit: the leak check sees every staging buffer freed


def test_host_staging_freed_by_destroy():
    """aqua_destroy releases the copy-engine staging buffers: contexts that
    page to host DRAM through the copy engines do not leak device memory."""
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    free0 = torch.cuda.mem_get_info()[0]
    for it in range(4):
        rig = Rig(L=2, bs=16, H=2, D=64, NB=16, lender_slots=0, host_slots=8, seed=it)
        rig.ctx.set_option(aqua.OPT_KERNEL, aqua.KERNEL_CE_HOST)
        rig.ctx.alloc_blocks(1, 4)
        rig.opool.alloc_blocks(1, 4)
        rig.ctx.swap_out([1])
        rig.opool.swap_out([1])
        rig.ctx.swap_in([1])
        rig.opool.swap_in([1])
        rig.assert_bytes_equal("ce round trip")
        rig.ctx.close()
        del rig
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 < (256 << 20), (free0, free1)


@pytest.mark.parametrize("engine", ["auto", "tma_dyn1", "tma_hybrid", "auto_staged"])
@pytest.mark.parametrize("seed", list(range(max(3, len(FUZZ_SEEDS)))))
def test_multistream_fuzz_equals_sequential(seed, engine, monkeypatch):
    """R7 end to end: random library ops (fills, swaps, migrations, prefix
    store/load, frees), each on a random one of three streams, must leave
    exactly the bytes of the oracle's sequential execution -- every reuse
    of a block or slot is ordered by the library's tickets (and, with
    claimed batches, every reuse of a launch counter pair)."""
    from oracle import pattern as opat
    rnd = random.Random(100 + seed)
    if engine == "auto_staged":
        # every call's descriptors through the pinned staging ring, which starts at 256 B so that it wraps
        # (host-waiting on the regions still in flight on other streams) and regrows within a few calls
        monkeypatch.setenv("AQUA_STAGE_MIN_BYTES", "256")
    rig = Rig(L=3, bs=16, H=2, D=64, NB=64, lender_slots=24, host_slots=24, seed=seed)
    c, o = rig.ctx, rig.opool
    if engine == "auto_staged":
        c.set_option(aqua.OPT_INLINE_MAX, 0)
    elif engine != "auto":
        _engine(c, engine)
    streams = [torch.cuda.Stream() for _ in range(3)]
    ntok = {}
    pids = list(range(6))
    for step in range(120):
        st = rnd.choice(streams).cuda_stream
        k = rnd.random()
        p = rnd.choice(pids)
        try:
            if k < 0.25:
                n = rnd.randint(1, 4)
                ids = o.alloc_blocks(p, n)
                assert c.alloc_blocks(p, n, st) == ids
                t0 = ntok.get(p, 0)
                t1 = len(o.prompts[p].blocks) * 16
                opat.write_tokens(o, p, t0, t1, 7)
                c.kv_fill_pattern(p, t0, t1, 7, st)
                ntok[p] = t1
            elif k < 0.45:
                sel = rnd.sample(pids, rnd.randint(1, 3))
                o.swap_out(sel)
                c.swap_out(sel, st)
            elif k < 0.65:
                sel = rnd.sample(pids, rnd.randint(1, 3))
                want = o.swap_in(sel)
                assert c.swap_in(sel, st)[0] == want
            elif k < 0.72:
                dst = rnd.choice([kp.LOC_PEER, kp.LOC_HOST])
                o.migrate([p], dst)
                c.migrate([p], dst, st)
            elif k < 0.78:
                f = rnd.randint(0, 1)
                n = rnd.randint(0, 3)
                o.prefix_store(f, p, n)
                c.prefix_store(f, p, n, st)
            elif k < 0.84:
                f = rnd.randint(0, 1)
                want = o.prefix_load(f, p)
                assert c.prefix_load(f, p, st)[0] == want
            elif k < 0.88:
                f = rnd.randint(0, 1)
                o.prefix_drop(f)
                c.prefix_drop(f)
            else:
                o.free_prompt(p)
                c.free(p, st)
                ntok.pop(p, None)
        except kp.AquaError:
            continue      # the oracle refused: the library must not have been called
        if step % 40 == 39:
            rig.assert_bytes_equal(f"fuzz step {step}")
    rig.assert_bytes_equal("fuzz end")


@pytest.mark.parametrize("pieces", [1, 3, 8])
@pytest.mark.parametrize("arena", ["lender", "lender_dyn", "host", "host_ce"])
def test_swap_exchange_bytes(pieces, arena):
    """aqua_swap_exchange == swap_out then swap_in (oracle), byte for byte,
    with the resume on another stream pipelined behind the preemption pieces
    whose blocks it reuses ("lender_dyn": both directions' kernels claim
    1-unit batches from their own counters while they run concurrently)."""
    rig = Rig(L=3, bs=16, H=4, D=64, NB=40, lender_slots=30 if arena in ("lender", "lender_dyn") else 0,
              host_slots=40)
    c, o = rig.ctx, rig.opool
    if arena == "host_ce":
        c.set_option(aqua.OPT_KERNEL, aqua.KERNEL_CE_HOST)
    if arena == "lender_dyn":
        c.set_option(aqua.OPT_TMA_SCHED, 1)
        c.set_option(aqua.OPT_TMA_PIECE, 4096)        # S = 8 KiB -> 2 pieces per chunk, many units
    perm = block_permutation(40, 40, seed=11).tolist()
    for pid, k in ((1, 6), (2, 5), (3, 7), (4, 9)):
        ids, perm = perm[:k], perm[k:]
        c.adopt_blocks(pid, ids)
        o.adopt_blocks(pid, ids)
    _ops(rig, [("out", [2, 4])])
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    new, to, ti = c.swap_exchange([1, 3], [4, 2], s1.cuda_stream, s2.cuda_stream, pieces=pieces)
    o.swap_out([1, 3])
    assert new == o.swap_in([4, 2])
    rig.assert_bytes_equal("exchange")
    # and back again, same streams swapped
    new, to, ti = c.swap_exchange([4], [1, 3], s2.cuda_stream, s1.cuda_stream, pieces=pieces)
    o.swap_out([4])
    assert new == o.swap_in([1, 3])
    rig.assert_bytes_equal("exchange back")


def test_swap_exchange_timing_spans_pieces():
    rig = Rig(L=4, bs=16, H=8, D=128, NB=96, lender_slots=96)
    c = rig.ctx
    c.alloc_blocks(1, 32)
    c.alloc_blocks(2, 32)
    c.swap_out([2])
    c.set_option(aqua.OPT_TIMING, 1)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    _, to, ti = c.swap_exchange([1], [2], s1.cuda_stream, s2.cuda_stream, pieces=4)
    torch.cuda.synchronize()
    t_one = c.swap_out([2], s1.cuda_stream)    # pid 2 is resident again; time a plain swap of the same size
    torch.cuda.synchronize()
    assert c.ticket_elapsed(to) > 0.5 * c.ticket_elapsed(t_one)
    assert c.ticket_elapsed(ti) > 0


def test_library_owned_lender_reclaim_frees_after_ticket():
    """aqua_lend(base=NULL) allocates the lender arena itself; a reclaim
    moves the images to the host and frees the arena once its ticket is
    done (deferred free); the images stay byte-exact (verify after resume)."""
    import torch
    L, bs, H, D, NB = 4, 16, 8, 128, 64
    S = bs * H * D * 2
    layers = [torch.zeros(2 * NB * S, dtype=torch.uint8, device="cuda") for _ in range(L)]
    c = aqua.Ctx(0, L, bs, H, D, 2, NB, [t.data_ptr() for t in layers])
    U = c.U
    assert c.lend(0, 0, 40 * U) == 40
    assert c.lend(aqua.HOST, 0, 40 * U) == 40
    base, n = c.arena_base(aqua.LOC_PEER)
    assert base and n == 40
    c.alloc_blocks(1, 16)
    c.alloc_blocks(2, 8)
    c.kv_fill_pattern(1, 0, 16 * bs, 5)
    c.kv_fill_pattern(2, 0, 8 * bs, 5)
    c.swap_out([1, 2])
    t = c.reclaim()
    c.sync(t)
    assert c.counts()[1] == -1 and c.query(1)[1] == aqua.LOC_HOST
    for x in layers:
        x.fill_(0x33)
    c.swap_in([2, 1])
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    c.kv_verify_pattern(1, 16 * bs, 5, cnt.data_ptr())
    c.kv_verify_pattern(2, 8 * bs, 5, cnt.data_ptr())
    torch.cuda.synchronize()
    assert int(cnt.item()) == 0
    c.alloc_blocks(3, 1)          # a later call retires the ticket and frees the zombie arena
    assert c.lend(0, 0, 8 * U) == 8   # re-offer: a fresh library-owned arena
    c.close()


def test_pattern_batch_kernel_matches_oracle_words():
    rig = Rig(L=2, bs=16, H=2, D=64, NB=16, lender_slots=0)
    for pid, ids in ((3, [6, 2]), (4, [9]), (5, [0, 12, 1])):
        rig.ctx.adopt_blocks(pid, ids)
        rig.opool.adopt_blocks(pid, ids)
    rig.ctx.kv_fill_pattern_batch([3, 4, 5], [5, 0, 17], [27, 16, 40], 99)
    for pid, t0, t1 in ((3, 5, 27), (4, 0, 16), (5, 17, 40)):
        opat.write_tokens(rig.opool, pid, t0, t1, 99)
    rig.assert_bytes_equal("pattern batch")


@pytest.mark.parametrize("engine", KERNEL_ENGINES)
def test_many_small_blocks_whole_buffer(engine):
    """Scale edge: 131,072 blocks of S = 256 B (100,000-block prompt, 800 KB of
    staged descriptors, slot ids > 2^16), whole pool / arena compared with
    the oracle after swap_out and after swap_in into a fragmented pool."""
    NB = 131072
    rig = Rig(L=1, bs=16, H=1, D=8, NB=NB, lender_slots=100000, host_slots=0)
    c, o = rig.ctx, rig.opool
    _engine(c, engine)
    perm = block_permutation(NB, NB, seed=13).tolist()
    _ops(rig, [("adopt", (1, perm[:100000])), ("adopt", (2, perm[100000:100500])), ("out", [1]),
               ("alloc", (3, 20000)), ("in", [1])])


def test_dynamic_schedule_counter_reuse_across_streams():
    """Dynamically scheduled TMA launches claim batches through one of 256
    per-context counter pairs; 600 launches on three streams cycle through
    every pair more than twice (a pair is reused only after its last launch's
    ticket), and the bytes still equal the oracle's sequential execution."""
    rig = Rig(L=2, bs=16, H=2, D=64, NB=96, lender_slots=64, host_slots=0, seed=3)
    c, o = rig.ctx, rig.opool
    c.set_option(aqua.OPT_KERNEL, aqua.KERNEL_TMA)
    c.set_option(aqua.OPT_TMA_SCHED, 1)
    c.set_option(aqua.OPT_MAX_CTAS, 5)
    streams = [torch.cuda.Stream() for _ in range(3)]
    for p in range(6):
        assert c.alloc_blocks(p, 5) == o.alloc_blocks(p, 5)
    rnd = random.Random(7)
    n0 = c.launch_count()
    for step in range(300):
        sel = rnd.sample(range(6), rnd.randint(1, 3))
        c.swap_out(sel, rnd.choice(streams).cuda_stream)
        o.swap_out(sel)
        assert c.swap_in(sel, rnd.choice(streams).cuda_stream)[0] == o.swap_in(sel)
    assert c.launch_count() - n0 == 600
    rig.assert_bytes_equal("600 dynamically scheduled launches")


def test_auto_policy_launch_shapes():
    """aqua_last_launch reports what AUTO chose: claimed
    2-unit batches with a 4-stage ring at one CTA per SM; static ranges for a
    small call; under an SM cap, static ranges for stage-sized chunks and the
    hybrid ring + LDST warps for sub-stage chunks of 2 KiB and up, the
    small-chunk kernel (16-warp CTAs) for 512 B / 1 KiB; at full grid the batch
    size by chunk size, and the small-chunk kernel for 512 B / 1 KiB chunks."""
    def ctx_for(L, H, NB, nslots, D=128):
        S = 16 * H * D * 2
        layers = [torch.zeros(2 * NB * S, dtype=torch.uint8, device="cuda") for _ in range(L)]
        arena = torch.zeros(nslots * 2 * L * S, dtype=torch.uint8, device="cuda")
        c = aqua.Ctx(0, L, 16, H, D, 2, NB, [t.data_ptr() for t in layers])
        c.lend(0, arena.data_ptr(), arena.numel())
        return c, layers, arena

    c, keep, arena = ctx_for(4, 8, 2600, 2600)            # S = 32 KiB: one chunk per stage
    with pytest.raises(aqua.AquaError):
        c.last_launch()
    c.alloc_blocks(1, 2500)
    c.swap_out([1])
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    s = c.last_launch()
    assert s["engine"] == "tma" and s["variant"] == 0 and s["ctas"] == sm and s["stages"] == 4
    assert s["schedule"] == "claimed batches of 2 items" and s["inline_descriptors"] == 2500
    c.swap_in([1])
    c.alloc_blocks(2, 3)                                   # small call: static ranges
    c.swap_out([2])
    assert c.last_launch()["schedule"] == "static ranges"
    c.set_option(aqua.OPT_MAX_CTAS, 16)
    c.swap_out([1])
    s = c.last_launch()
    assert s["ctas"] == 16 and s["variant"] == 0 and s["schedule"] == "static ranges"
    c.swap_in([1])
    c.set_option(aqua.OPT_MAX_CTAS, 0)
    c.set_option(aqua.OPT_RATE_GBPS, 420)                 # budget -> ceil(420 / 50) = 9 SMs
    c.swap_out([1])
    assert c.last_launch()["ctas"] == 9
    c.set_option(aqua.OPT_MAX_CTAS, 4)                    # the smaller cap wins
    c.swap_in([1])
    assert c.last_launch()["ctas"] == 4
    c.close()
    del keep, arena

    c, keep, arena = ctx_for(8, 2, 2600, 2600)            # S = 8 KiB: 4 chunks per stage
    c.alloc_blocks(1, 2500)
    c.set_option(aqua.OPT_MAX_CTAS, 16)
    c.swap_out([1])
    s = c.last_launch()
    assert s["ctas"] == 16 and s["variant"] == 3 and s["threads_per_cta"] == 288
    assert s["schedule"] == "claimed batches of 128 items"  # the ring's 32 units x 4 chunks
    c.swap_in([1])
    c.close()
    del keep, arena

    # sub-stage chunks at full grid (round 2, profiles/r02_small_chunks_*.jsonl, r02_small_ldst2.jsonl):
    # 2 KiB -> ring, 4-unit batches; 1 KiB and 512 B -> the small-chunk register kernel, 2 CTAs per SM
    for D, engine, variant, sched in ((64, "tma", 0, "claimed batches of 64 items"), (32, "ldst", 3, "static ranges"),
                                      (16, "ldst", 3, "static ranges")):
        c, keep, arena = ctx_for(32, 1, 5000, 5000, D=D)
        c.alloc_blocks(1, 5000)
        c.swap_out([1])
        s = c.last_launch()
        assert s["engine"] == engine and s["variant"] == variant, (D, s)
        assert s["ctas"] == (sm if engine == "tma" else 2 * sm) and s["schedule"] == sched, (D, s)
        assert s["threads_per_cta"] == {(0, "tma"): 32, (3, "tma"): 288, (3, "ldst"): 256}[(variant, engine)]
        c.swap_in([1])
        # under an SM cap (r02_small_caps.jsonl): 512 B and 1 KiB -> the small-chunk kernel with 16-warp
        # CTAs, one per allowed SM; 2 KiB -> the hybrid ring + register warps
        c.set_option(aqua.OPT_MAX_CTAS, 24)
        c.swap_out([1])
        s = c.last_launch()
        if D == 64:
            assert (s["engine"], s["variant"], s["ctas"], s["threads_per_cta"]) == ("tma", 3, 24, 288), s
        else:
            assert (s["engine"], s["variant"], s["ctas"], s["threads_per_cta"]) == ("ldst", 3, 24, 512), s
        c.swap_in([1])
        c.close()
        del keep, arena


@pytest.mark.parametrize("shape", ["s512", "s1k"])
@pytest.mark.parametrize("ctas", [3, 0])
def test_hybrid_register_warps_packed_chunks_at_scale(shape, ctas):
    """The hybrid's register warps pack whole 512 B / 1 KiB chunks into 4 KiB
    rounds (AUTO runs this for capped launches on a peer arena).  The small
    random sequences leave those warps little to claim, so this call is big
    enough (6,000 blocks on a fragmented pool) that they claim most batches;
    whole pool and arena equal the oracle after swap_out and after swap_in."""
    L, bs, H, D = SHAPES[shape][:4]
    NB = 8192
    rig = Rig(L=L, bs=bs, H=H, D=D, NB=NB, lender_slots=6500, host_slots=0)
    c, o = rig.ctx, rig.opool
    _engine(c, "tma_hybrid")
    c.set_option(aqua.OPT_MAX_CTAS, ctas)
    perm = block_permutation(NB, NB, seed=29).tolist()
    _ops(rig, [("adopt", (1, perm[:6000])), ("adopt", (2, perm[6000:6100])), ("out", [1]),
               ("alloc", (3, 1500)), ("in", [1])])


@pytest.mark.parametrize("late", ["migrate", "none"])
def test_migration_source_slots_reused_on_another_stream(late):
    """R7 for NEXT-1: a migration reads the image's old slots; they are free
    the moment aqua_migrate returns, and a swap_out on another stream lands
    in them (lowest free slots).  With the migration delayed by a ~20 ms sleep
    on its stream, the swap_out must still wait for it (the freed slots carry
    the migration's ticket).  Whole buffers must equal the oracle's
    sequential run."""
    L, bs, H, D, NB = 4, 16, 8, 128, 64          # U = 256 KiB
    rig = Rig(L=L, bs=bs, H=H, D=D, NB=NB, lender_slots=24, host_slots=24)
    c, o = rig.ctx, rig.opool
    s_mig, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    for p in range(3):
        assert c.alloc_blocks(p, 8) == o.alloc_blocks(p, 8)
    _ops(rig, [("out", [0])])                     # image of 0 on lender slots 0..7
    torch.cuda.synchronize()
    if late == "migrate":
        with torch.cuda.stream(s_mig):
            torch.cuda._sleep(40_000_000)
    c.migrate([0], aqua.LOC_HOST, s_mig.cuda_stream)
    o.migrate([0], kp.LOC_HOST)
    c.swap_out([1], s_out.cuda_stream)            # -> lender slots 0..7 again
    o.swap_out([1])
    rig.assert_bytes_equal(f"migration source reuse, late {late}")


@pytest.mark.parametrize("engine", ["auto", "ce_host"])
def test_copy_engine_staging_shared_by_two_streams(engine):
    """The copy-engine host path stages every host-bound call through one GPU
    buffer per direction.  A large swap_out (64 MiB: ~1.2 ms of PCIe DMA out
    of the buffer) on one stream and a second swap_out right after on another
    stream: the second call's gather into the buffer must wait until the
    first call's DMA has read it.  Whole buffers equal the oracle's."""
    L, bs, H, D, NB = 32, 16, 8, 128, 96         # U = 2 MiB (Llama-3-8B block)
    rig = Rig(L=L, bs=bs, H=H, D=D, NB=NB, lender_slots=0, host_slots=80)
    c, o = rig.ctx, rig.opool
    _engine(c, engine)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    assert c.alloc_blocks(1, 32) == o.alloc_blocks(1, 32)
    assert c.alloc_blocks(2, 32) == o.alloc_blocks(2, 32)
    torch.cuda.synchronize()
    # the two library calls back to back (the oracle's copies would give the GPU time to finish the first)
    c.swap_out([1], s1.cuda_stream)
    c.swap_out([2], s2.cuda_stream)
    o.swap_out([1])
    o.swap_out([2])
    rig.assert_bytes_equal(f"two host swap_outs on two streams, {engine}")
    new1, _ = c.swap_in([1], s1.cuda_stream)
    new2, _ = c.swap_in([2], s2.cuda_stream)
    assert new1 == o.swap_in([1])
    assert new2 == o.swap_in([2])
    rig.assert_bytes_equal(f"two host swap_ins on two streams, {engine}")


@pytest.mark.parametrize("late", ["store", "load"])
def test_prefix_cache_reuse_with_a_delayed_stream(late):
    """R7 for NEXT-2, made deterministic with a ~20 ms sleep:
      store -- a delayed prefix_store reads the source prompt's blocks; the
               prompt is freed and its blocks reallocated and overwritten on
               another stream right away: the overwrite must wait for the
               store (the blocks carry its ticket);
      load  -- a delayed prefix_load reads the cached image; the prefix is
               dropped and a swap_out on another stream lands in its slots:
               the swap_out must wait for the load.
    Whole buffers equal the oracle's sequential run."""
    L, bs, H, D, NB = 4, 16, 8, 128, 64          # U = 256 KiB
    rig = Rig(L=L, bs=bs, H=H, D=D, NB=NB, lender_slots=16, host_slots=0)
    c, o = rig.ctx, rig.opool
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    assert c.alloc_blocks(5, 8) == o.alloc_blocks(5, 8)
    assert c.alloc_blocks(8, 6) == o.alloc_blocks(8, 6)
    torch.cuda.synchronize()
    if late == "store":
        with torch.cuda.stream(s1):
            torch.cuda._sleep(40_000_000)
    c.prefix_store(9, 5, 8, s1.cuda_stream)
    o.prefix_store(9, 5, 8)
    if late == "store":
        c.free(5, s2.cuda_stream)
        o.free_prompt(5)
        ids = c.alloc_blocks(6, 8, s2.cuda_stream)
        assert ids == o.alloc_blocks(6, 8)
        with torch.cuda.stream(s2):
            for l in range(L):
                for kv in (0, 1):
                    for b in ids:
                        off = kv * rig.lay.P_kv + b * rig.lay.P_b
                        rig.layers[l][off:off + rig.lay.S].fill_(0x5A)
                        o.chunk(l, kv, b)[:] = 0x5A
        torch.cuda.synchronize()
        new, _ = c.prefix_load(9, 7)
        assert new == o.prefix_load(9, 7)
    else:
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            torch.cuda._sleep(40_000_000)
        new, _ = c.prefix_load(9, 7, s1.cuda_stream)
        assert new == o.prefix_load(9, 7)
        c.prefix_drop(9)
        o.prefix_drop(9)
        c.swap_out([8], s2.cuda_stream)          # -> the dropped image's slots 0..5
        o.swap_out([8])
    rig.assert_bytes_equal(f"prefix reuse, late {late}")


def test_exchange_resume_waits_for_the_piece_that_frees_its_blocks():
    """aqua_swap_exchange pipelines the resume behind the preemption pieces:
    each resume descriptor waits for the piece that reads the block it
    reuses.  Deterministic setup: the preempted prompt A (48 x 2 MiB) goes to
    host DRAM (PCIe: each of the 3 pieces takes ~0.6 ms) while the resumed
    prompt B comes from the lender (HBM: microseconds); A's block table runs
    from the highest ids down, so B's fresh blocks (lowest-first) are the
    ones the LAST piece reads.  Resuming after the first piece only would
    overwrite them before they reach DRAM.  Whole buffers equal the
    oracle's swap_out-then-swap_in."""
    L, bs, H, D, NB = 32, 16, 8, 128, 64         # U = 2 MiB
    rig = Rig(L=L, bs=bs, H=H, D=D, NB=NB, lender_slots=16, host_slots=48)
    c, o = rig.ctx, rig.opool
    assert c.alloc_blocks(2, 16) == o.alloc_blocks(2, 16)      # B: blocks 0..15
    a_ids = list(range(NB - 1, 15, -1))                          # A: 63 .. 16
    c.adopt_blocks(1, a_ids)
    o.adopt_blocks(1, a_ids)
    _ops(rig, [("out", [2])])                                    # B -> the lender (now full)
    _ops(rig, [("alloc", (3, 16))])                              # filler: no free block left
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    new, _, _ = c.swap_exchange([1], [2], s1.cuda_stream, s2.cuda_stream, pieces=3)
    o.swap_out([1])
    assert new == o.swap_in([2]) == [list(range(16, 32))]
    assert c.query(1)[1] == aqua.LOC_HOST
    rig.assert_bytes_equal("exchange, resume into the last piece's blocks")


def test_descriptor_ring_reuse_with_a_delayed_stream(monkeypatch):
    """Staged descriptors (inline tier off) through a ring of a few regions:
    a swap_out on a stream held back by a ~20 ms sleep has its descriptor
    upload still queued when a second call on another stream wraps the ring
    onto the same region.  The library must wait (host) for the region's
    last user before rewriting it; otherwise the delayed call would move the
    second call's blocks.  Whole buffers equal the oracle's."""
    monkeypatch.setenv("AQUA_STAGE_MIN_BYTES", "256")
    L, bs, H, D, NB = 2, 16, 2, 64, 64          # S = 4 KiB
    rig = Rig(L=L, bs=bs, H=H, D=D, NB=NB, lender_slots=64, host_slots=0)
    c, o = rig.ctx, rig.opool
    c.set_option(aqua.OPT_INLINE_MAX, 0)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    perm = block_permutation(NB, NB, seed=5).tolist()
    for pid in range(4):                          # 16 blocks each: 128 B of descriptors per call
        ids = perm[16 * pid:16 * (pid + 1)]
        c.adopt_blocks(pid, ids)
        o.adopt_blocks(pid, ids)
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        torch.cuda._sleep(40_000_000)
    c.swap_out([0], s1.cuda_stream)               # its upload waits behind the sleep
    for pid in (1, 2, 3):                         # the ring (256 B: two regions) wraps onto its region
        c.swap_out([pid], s2.cuda_stream)
    for pid in range(4):
        o.swap_out([pid])
    rig.assert_bytes_equal("staged descriptors, delayed first call")


@pytest.mark.parametrize("engine", ["tma", "ldst"])
def test_zero_copy_host_launches_are_capped(engine):
    """A zero-copy swap whose images all live in pinned host DRAM is bound by
    PCIe (~55 GB/s), which 8 CTAs saturate; AUTO's policy caps such launches
    at 8 CTAs and leaves the other SMs to decode (DESIGN 5.1).  A launch that
    also touches HBM images is not capped."""
    rig = Rig(L=4, bs=16, H=8, D=128, NB=64, lender_slots=8, host_slots=40)
    c, o = rig.ctx, rig.opool
    _engine(c, engine)
    _ops(rig, [("alloc", (1, 8)), ("alloc", (2, 20)), ("out", [1]), ("out", [2])])   # 1 -> lender, 2 -> host
    assert c.query(2)[1] == aqua.LOC_HOST
    assert c.last_launch()["ctas"] <= 16                       # host-only launch: 8 CTAs (LDST: 2 x 8)
    _ops(rig, [("in", [2])])
    assert c.last_launch()["ctas"] <= 16
    _ops(rig, [("in", [1])])
    assert c.last_launch()["ctas"] > 16                        # lender images: the whole GPU


@pytest.mark.parametrize("engine", ["auto", "tma", "tma_hybrid", "ldst", "ldst_small"])
def test_degenerate_and_maximum_calls_bytes(engine):
    """The method's degenerate and maximum cases in one context, whole pool
    and both arenas compared with the oracle after every call (R4, R5):
    empty calls; a prompt that owns no block; the whole pool paged out in ONE
    call into a lender with exactly NB slots; the next whole-pool prompt
    falling back to a host arena of exactly NB slots (lender full); a prompt
    that fits nowhere (NOSPACE); resumes needing one block more than is free
    (NOBLOCKS) and then exactly every free block.  A failed call must leave
    every byte and the bookkeeping as they were, with the oracle's code."""
    NB = 24
    rig = Rig(L=3, bs=16, H=1, D=32, NB=NB, lender_slots=NB, host_slots=NB, seed=7)   # S = 1 KiB, U = 6 KiB
    _engine(rig.ctx, engine)
    c, o = rig.ctx, rig.opool

    def fails(name, arg, code):
        with pytest.raises(kp.AquaError) as eo:
            {"alloc": lambda: o.alloc_blocks(*arg), "out": lambda: o.swap_out(arg),
             "in": lambda: o.swap_in(arg)}[name]()
        with pytest.raises(aqua.AquaError) as ec:
            {"alloc": lambda: c.alloc_blocks(*arg), "out": lambda: c.swap_out(arg),
             "in": lambda: c.swap_in(arg, cap=4 * NB)}[name]()
        assert eo.value.code == ec.value.code == code, (name, arg, eo.value.code, ec.value.code)
        assert c.counts() == (len(o.free), len(o.peer.free), len(o.host.free))
        rig.assert_bytes_equal(f"after failed {name} {arg}")

    n0 = c.launch_count()
    _ops(rig, [("out", []), ("in", []), ("alloc", (9, 0)), ("out", [9]), ("in", [9]), ("free", 9)])
    assert c.launch_count() == n0                       # nothing to copy: no launch
    # three ragged prompts own the whole pool; one call pages all of it into the lender (exactly full)
    _ops(rig, [("alloc", (1, 1)), ("alloc", (2, 7)), ("alloc", (3, NB - 8)), ("out", [3, 1, 2])])
    assert c.counts() == (NB, 0, NB)
    # a fourth whole-pool prompt: the lender is full, so its image goes to the host arena (exactly full)
    _ops(rig, [("alloc", (4, NB)), ("out", [4])])
    assert c.query(4)[1] == aqua.LOC_HOST and c.counts() == (NB, 0, 0)
    _ops(rig, [("alloc", (5, 1))])
    fails("out", [5], aqua.E_NOSPACE)                   # fits nowhere
    fails("in", [4], aqua.E_NOBLOCKS)                   # needs NB blocks, NB - 1 are free
    fails("in", [3, 1, 2], aqua.E_NOBLOCKS)             # the same, over three images in one call
    _ops(rig, [("in", [3, 2])])                         # needs exactly every free block (NB - 1)
    assert c.counts() == (0, NB - 1, 0)
    _ops(rig, [("free", 5), ("in", [1])])               # the pool is full again
    assert c.counts() == (0, NB, 0)
    fails("alloc", (6, 1), aqua.E_NOBLOCKS)
    _ops(rig, [("free", 3), ("free", 1), ("free", 2), ("in", [4]), ("out", [4])])
    assert c.query(4)[1] == aqua.LOC_PEER and c.counts() == (NB, 0, NB)   # lowest arena with room (R5)
    _ops(rig, [("in", [4])])
    assert c.counts() == (0, NB, NB)


@pytest.mark.parametrize("nblk", [3, 300])
def test_mixed_arena_call_split_bytes(nblk):
    """AUTO splits a call whose images land in both arenas (the lender fills
    up, R5): the lender images on the TMA kernel, the host ones through the
    copy engines, on the same stream.  Whole buffers vs the oracle after the
    mixed swap_out and the mixed swap_in; 300 blocks per prompt put the
    descriptors of both parts beyond the inline tier (staged uploads)."""
    NB = 4 * nblk + 8
    rig = Rig(L=2, bs=16, H=1, D=64, NB=NB, lender_slots=nblk + 1, host_slots=2 * nblk, seed=3)
    c = rig.ctx
    c.set_option(aqua.OPT_INLINE_MAX, 256)
    _ops(rig, [("alloc", (1, nblk)), ("alloc", (2, 1)), ("alloc", (3, nblk)), ("alloc", (4, 5))])
    n0 = c.launch_count()
    _ops(rig, [("out", [1, 3, 2])])
    assert (c.query(1)[1], c.query(3)[1], c.query(2)[1]) == (aqua.LOC_PEER, aqua.LOC_HOST, aqua.LOC_PEER)
    # two launches: the lender part on the TMA kernel, the copy engines' gather of the host part
    # (one fused launch would hold every SM for the PCIe time: profiles/r02_mixed_split.jsonl)
    assert c.launch_count() - n0 == 2
    _ops(rig, [("in", [3, 1]), ("out", [3]), ("in", [2, 3]), ("free", 1), ("free", 4)])
    assert c.query(3)[0] == aqua.RESIDENT
    c.set_option(aqua.OPT_KERNEL, aqua.KERNEL_TMA)      # an explicit engine: one fused launch
    _ops(rig, [("alloc", (5, nblk + 1)), ("out", [3, 5])])
    n0 = c.launch_count()
    _ops(rig, [("in", [5, 3])])
    assert c.launch_count() - n0 == 1


@pytest.mark.parametrize("layer_group", [1, 3])
@pytest.mark.parametrize("nblk", [4, 300])
def test_layerwise_mixed_arena_split_bytes(layer_group, nblk):
    """NEXT-3 with a call whose images span lender and host: AUTO splits
    every layer group (no shared descriptor upload), one ticket per group;
    whole buffers vs the oracle."""
    rig = Rig(L=4, bs=16, H=2, D=32, NB=3 * nblk + 8, lender_slots=nblk, host_slots=nblk, seed=5)
    c, o = rig.ctx, rig.opool
    c.set_option(aqua.OPT_INLINE_MAX, 256)
    for pid in (1, 2):
        assert c.alloc_blocks(pid, nblk) == o.alloc_blocks(pid, nblk)
    n0 = c.launch_count()
    tks = c.swap_out_layers([1, 2], layer_group)
    o.swap_out([1, 2])
    ng = -(-4 // layer_group)
    assert len(tks) == ng and tks == sorted(tks) and c.launch_count() - n0 == 2 * ng
    assert (c.query(1)[1], c.query(2)[1]) == (aqua.LOC_PEER, aqua.LOC_HOST)
    rig.assert_bytes_equal("layered mixed swap_out")
    assert c.alloc_blocks(3, 5) == o.alloc_blocks(3, 5)
    new, tks = c.swap_in_layers([2, 1], layer_group)
    assert new == o.swap_in([2, 1]) and len(tks) == ng
    rig.assert_bytes_equal("layered mixed swap_in")


@pytest.mark.parametrize("engine", ["auto", "tma"])
def test_migration_runs_with_fragmented_slots_bytes(engine):
    """NEXT-1 migration moves runs of slots that are consecutive on BOTH
    sides as one copy (AUTO: one DMA): consecutive source slots whose lowest
    free destination slots have a hole (and the reverse) must split into
    runs.  Whole buffers vs the oracle after every call."""
    rig = Rig(L=2, bs=16, H=2, D=64, NB=24, lender_slots=8, host_slots=8, seed=11)
    c, o = rig.ctx, rig.opool
    _engine(c, engine)

    def mig(pids, dst):
        c.migrate(pids, dst)
        o.migrate(pids, {aqua.LOC_PEER: kp.LOC_PEER, aqua.LOC_HOST: kp.LOC_HOST}[dst])
        rig.assert_bytes_equal(f"migrate {pids} -> {dst}")

    _ops(rig, [("alloc", (1, 1)), ("alloc", (2, 1)), ("alloc", (3, 1)), ("alloc", (4, 4)), ("out", [1, 2, 3])])
    mig([1, 2, 3], aqua.LOC_HOST)                       # lender 0..2 -> host 0..2
    mig([2], aqua.LOC_PEER)                             # host slot 1 becomes a hole
    _ops(rig, [("out", [4])])                           # lender 1..4
    mig([4], aqua.LOC_HOST)                             # consecutive source -> host 1, 3, 4, 5
    assert c.query(4, with_ids=True)[3] == [1, 3, 4, 5]
    mig([1], aqua.LOC_PEER)                             # host slot 0 becomes a hole: lender 1
    mig([4, 3], aqua.LOC_PEER)                          # host 1, 3, 4, 5 then 2 -> lender 2..6
    _ops(rig, [("in", [4, 3, 2, 1])])
