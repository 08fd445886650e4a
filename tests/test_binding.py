"""The ctypes binding's hot calls marshal through per-Ctx scratch buffers
(paper_2407_21255_b200/aqua.py).  These dry-run tests (no GPU) pin what the
scratch must not change: results are copies, not views of the scratch;
calls of many prompts grow it; a swap_in needing more ids than the pool has
still reports the library's own error (pool exhausted, not "out_ids too
small"); and the results equal a fresh-array marshalling of the same call."""
import pytest

from paper_2407_21255_b200 import aqua


def _ctx(NB=100, slots=400, L=2):
    c = aqua.Ctx(aqua.DRYRUN, L, 16, 1, 16, 2, NB, [(l + 1) << 40 for l in range(L)])
    c.lend(0, 8 << 40, slots * c.U)
    return c


def test_results_are_copies():
    c = _ctx()
    a = c.alloc_blocks(1, 10)
    b = c.alloc_blocks(2, 10)
    assert a == list(range(10)) and b == list(range(10, 20))
    c.swap_out([1, 2])
    t1, _ = c.swap_in([2])
    t2, _ = c.swap_in([1])
    assert t1 == [list(range(10))] and t2 == [list(range(10, 20))]
    assert a == list(range(10)) and b == list(range(10, 20))      # earlier results untouched
    c.close()


def test_many_prompts_grow_scratch():
    c = _ctx(NB=400, slots=400)
    pids = list(range(1, 201))                                     # > the 64-entry initial scratch
    for p in pids:
        c.alloc_blocks(p, 2)
    c.swap_out(pids)
    tables, t = c.swap_in(pids[::-1])
    assert len(tables) == 200 and all(len(x) == 2 for x in tables)
    assert sorted(b for x in tables for b in x) == list(range(400))
    assert tables[0] == [0, 1] and tables[-1] == [398, 399]        # lowest-first in call order (R4)
    assert t > 0
    c.close()


def test_oversized_swap_in_reports_pool_exhausted():
    c = _ctx(NB=100, slots=400)
    c.alloc_blocks(1, 80)
    c.swap_out([1])
    c.alloc_blocks(2, 80)
    c.swap_out([2])
    with pytest.raises(aqua.AquaError) as e:                       # needs 160 ids > NB = 100
        c.swap_in([1, 2])
    assert e.value.code == aqua.E_NOBLOCKS
    with pytest.raises(aqua.AquaError) as e:
        c.swap_in([1, 1])
    assert e.value.code == aqua.E_INVAL and "duplicate" in str(e.value)
    with pytest.raises(aqua.AquaError) as e:
        c.swap_in([77])
    assert e.value.code == aqua.E_STATE
    c.close()


def test_explicit_cap_path_matches_scratch_path():
    res = []
    for cap in (-1, 64):
        c = _ctx()
        for p in (1, 2, 3):
            c.alloc_blocks(p, 5 + p)
        c.swap_out([3, 1])
        c.alloc_blocks(9, 4)
        res.append(c.swap_in([1, 3], cap=cap)[0])
        c.close()
    assert res[0] == res[1]


def test_exchange_through_scratch():
    c = _ctx()
    c.alloc_blocks(1, 6)
    c.alloc_blocks(2, 7)
    c.swap_out([2])
    tables, to, ti = c.swap_exchange([1], [2])
    assert [len(x) for x in tables] == [7] and to > 0 and ti > 0
    assert c.query(1)[0] == aqua.SWAPPED and c.query(2)[0] == aqua.RESIDENT
    c.close()


def test_swap_in_as_arrays_equals_lists():
    import numpy as np
    res = []
    for as_arrays in (False, True):
        c = _ctx(NB=60, slots=60)
        for p in (1, 2, 3):
            c.alloc_blocks(p, 3 + p)
        c.swap_out([1, 2, 3])
        c.alloc_blocks(9, 5)
        tables, _ = c.swap_in([3, 1, 2], as_arrays=as_arrays)
        if as_arrays:
            assert all(isinstance(t, np.ndarray) and t.dtype == np.int32 for t in tables)
            tables = [t.tolist() for t in tables]
        res.append(tables)
        c.close()
    assert res[0] == res[1] and [len(t) for t in res[0]] == [6, 4, 5]
