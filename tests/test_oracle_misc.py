"""Pins for oracle/pattern.py, oracle/bwfit.py and the seeded generators.

* splitmix64 against its published reference outputs (seed 0 sequence of
  Vigna's splitmix64: e220a8397b1dcdaf, 6e789e6aa1b965f4, 06c45d188009454f);
* the pattern's field packing is injective on the field ranges (distinct
  coordinates -> distinct packs) and a token write lands only in its row;
* SPEC's bandwidth-curve worked examples: (4 MB, 50 GB/s) and
  (64 MB, 200 GB/s) -> half 16 MB, peak 250 GB/s; B(320 MB) = 238.1 GB/s;
  320 MB in 160 buffers ~= 13.1 ms vs 1 buffer ~= 1.354 ms (10 us latency);
* generator determinism and SPEC's workload examples.
"""
import numpy as np
import pytest

from oracle import bwfit, pattern
from oracle import kvpool as kp
from workloads import block_permutation, burst_trace, kv_random_bytes, lognormal_lengths


def test_splitmix64_reference_vectors():
    g = 0x9E3779B97F4A7C15
    ref = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    xs = [0, g, (2 * g) % 2 ** 64]
    assert [pattern.splitmix64_int(x) for x in xs] == ref
    assert [int(v) for v in pattern.splitmix64(np.array(xs, dtype=np.uint64))] == ref


def test_pack_injective_on_field_ranges():
    rng = np.random.default_rng(5)
    n = 20000
    f = [rng.integers(0, 1 << w, n) for w in (16, 20, 8, 1, 7, 10)]
    packs = set()
    tuples = set()
    for p, t, l, kv, h, d in zip(*f):
        tuples.add((p, t, l, kv, h, d))
        packs.add(int(pattern.pack(int(p), int(t), int(l), int(kv), int(h), int(d))))
    assert len(packs) == len(tuples)


def test_write_tokens_touches_only_its_rows():
    lay = kp.Layout(L=2, bs=4, H=2, D=8, e=2, NB=6)
    layers = [np.zeros(lay.layer_bytes, np.uint8) for _ in range(2)]
    pool = kp.Pool(lay, layers)
    pool.adopt_blocks(3, [4, 1])
    pattern.write_tokens(pool, 3, 0, 5, seed=9)
    assert pattern.check_tokens(pool, 3, 5, seed=9)
    assert not pattern.check_tokens(pool, 3, 6, seed=9)   # token 5 unwritten
    # rows outside blocks 4 and 1 (and row >= 1 of block 1) stay zero
    for l in range(2):
        v = pool.layers[l].reshape(2, lay.NB, lay.bs, lay.H * lay.D * 2)
        for b in range(lay.NB):
            for i in range(lay.bs):
                written = (b == 4) or (b == 1 and i == 0)
                assert (v[:, b, i].any(axis=-1) == written).all() or not written
                if not written:
                    assert not v[:, b, i].any()
    # a different seed gives different words
    assert not pattern.check_tokens(pool, 3, 1, seed=10)


def test_bwfit_spec_examples():
    MB = 1e6
    peak, half = bwfit.calibrate(4 * MB, 50e9, 64 * MB, 200e9)
    assert peak == pytest.approx(250e9, rel=1e-12)
    assert half == pytest.approx(16 * MB, rel=1e-12)
    assert bwfit.effective_bandwidth(peak, half, 4 * MB) == pytest.approx(50e9, rel=1e-12)
    assert bwfit.effective_bandwidth(peak, half, 320 * MB) == pytest.approx(238.095e9, rel=1e-5)
    many = bwfit.transfer_time(peak, half, 320 * MB, 160, lat=10e-6)
    one = bwfit.transfer_time(peak, half, 320 * MB, 1, lat=10e-6)
    assert many == pytest.approx(13.12e-3, rel=1e-3)
    assert one == pytest.approx(1.354e-3, rel=1e-3)
    with pytest.raises(ValueError):
        bwfit.calibrate(1 * MB, 10e9, 2 * MB, 10e9)       # equal bandwidths
    # least squares recovers an exact curve
    sizes = [2 ** i * MB for i in range(8)]
    bws = [bwfit.effective_bandwidth(777e9, 3 * MB, s) for s in sizes]
    p2, h2 = bwfit.fit(sizes, bws)
    assert p2 == pytest.approx(777e9, rel=1e-9) and h2 == pytest.approx(3 * MB, rel=1e-9)
    # monotone and bounded by peak
    prev = 0
    for s in sizes:
        b = bwfit.effective_bandwidth(peak, half, s)
        assert prev <= b < peak
        prev = b


def test_generators_deterministic():
    assert np.array_equal(kv_random_bytes(1024, 0), kv_random_bytes(1024, 0))
    assert not np.array_equal(kv_random_bytes(1024, 0), kv_random_bytes(1024, 1))
    p = block_permutation(4096, 2048, seed=2)
    assert len(set(p.tolist())) == 2048 and p.max() < 4096
    assert burst_trace(seed=1) == burst_trace(seed=1)


def test_trace_shape():
    """Poisson count at 2.5/s x 60 s ~ 150; burst doubles it;
    medians of sharegpt-like lengths within 10%."""
    tr = burst_trace(seed=1)
    arr = np.array([a for _, a, _, _ in tr])
    t0 = arr[24]
    in_burst = ((arr > t0) & (arr < t0 + 60)).sum()
    assert 240 <= in_burst <= 360               # 2 x 2.5/s x 60 s = 300
    assert np.all(np.diff(arr) >= 0)
    rng = np.random.default_rng(0)
    x = lognormal_lengths(rng, 10000, 2000, 0.8, 1, 8192)
    assert abs(np.median(x) - 2000) / 2000 < 0.1 and x.max() <= 8192 and x.min() >= 1


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_write_token_range_equals_tokenwise_writes(seed):
    """The range writer (used by the bytes-mode trace replay) stores exactly
    the bytes of the token-by-token writer, for ranges that start and end
    mid-block on a scattered block table; nothing else in the pool moves."""
    rng = np.random.default_rng(seed)
    lay = kp.Layout(L=2, bs=16, H=2, D=8, e=2, NB=20)
    init = [kv_random_bytes(lay.layer_bytes, seed=s) for s in range(2)]
    a = kp.Pool(lay, [x.copy() for x in init])
    b = kp.Pool(lay, [x.copy() for x in init])
    ids = rng.permutation(20)[:9].tolist()
    a.adopt_blocks(4, ids)
    b.adopt_blocks(4, ids)
    t = 0
    while t < 9 * 16:
        n = int(rng.integers(1, 40))
        n = min(n, 9 * 16 - t)
        pattern.write_tokens(a, 4, t, t + n, seed=7)
        pattern.write_token_range(b, 4, t, t + n, seed=7)
        for l in range(2):
            assert np.array_equal(a.layers[l], b.layers[l]), (t, n)
        t += n
    assert pattern.check_tokens(b, 4, 9 * 16, seed=7)
    # one word against the scalar reference
    w = int(b.chunk(1, 1, ids[3])[(5 * 2 + 1) * 8 * 2 + 3 * 2:][:2].view(np.uint16)[0])
    want = pattern.splitmix64_int(7 ^ ((4 << 46) | ((3 * 16 + 5) << 26) | (1 << 18) | (1 << 17) | (1 << 10) | 3))
    assert w == want & 0xFFFF
