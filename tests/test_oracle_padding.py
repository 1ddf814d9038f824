"""Any n by "approach n from above" and the
diagonal-inclusive tetrahedron Delta_n^3 (i <= j <= k) run as the
strict set of n + 2 (reading E24).  Oracle pins: exact element covers against
the plain nested-loop enumerations for non-power-of-two n, the inclusive
triple rank against nested loops, and the C library's host-only plans (closed
forms, locate, rejected combinations).  CPU only."""
import itertools
import math

import numpy as np
import pytest


@pytest.mark.parametrize("n,want", [(1, 1), (2, 2), (3, 4), (5, 8), (1000, 1024), (1024, 1024), (1025, 2048)])
def test_padded_n(orc, n, want):
    assert orc.padded_n(n) == want


def test_rank3_inclusive_is_nested_loop_order(orc):
    n = 9
    pos = 0
    for k in range(n):
        for j in range(k + 1):
            for i in range(j + 1):
                assert orc.rank3_incl(i, j, k) == pos
                pos += 1
    assert pos == math.comb(n + 2, 3) == orc.domain_volume(3, True, n)
    np.testing.assert_array_equal(orc.index_write(3, True, n), np.arange(pos, dtype=np.uint32))
    # E24: rank3_incl(i, j, k) == rank3(i, j + 1, k + 2) (the strict set of n + 2)
    for i, j, k in itertools.combinations_with_replacement(range(7), 3):
        assert orc.rank3_incl(i, j, k) == orc.rank3(i, j + 1, k + 2)


@pytest.mark.parametrize("m,inc,n,rho", [(2, False, 1000, 16), (2, True, 1000, 16), (2, False, 33, 4), (2, True, 3, 2),
                                         (2, False, 130, 32), (3, False, 100, 4), (3, False, 67, 8), (3, True, 30, 2),
                                         (3, True, 61, 4), (3, False, 3, 1)])
@pytest.mark.parametrize("map_", ["lambda", "bb", "enum"])
def test_padded_element_cover_exact(orc, m, inc, n, rho, map_):
    nint = n + 2 if (m == 3 and inc) else n
    N = orc.padded_n(nint) // rho
    if map_ == "lambda" and ((m == 2 and N < 2) or (m == 3 and N < 8)):
        pytest.skip("grid below lambda's minimum")
    hits, r = orc.element_hits(m, inc, map_, n, rho)
    assert len(hits) == orc.domain_volume(m, inc, n)
    assert (hits == 1).all() and r["outside"] == 0
    assert r["useful"] == len(hits)
    assert r["launched"] == orc.grid_blocks(m, inc, map_, N) * rho ** m


def test_padded_thread_dump_brute_force(orc):
    # BB m=2, n = 6 on the grid of 8 (rho = 2): identity + filter j < i < n
    got = orc.thread_dump(2, False, "bb", 6, 2)
    exp = []
    for I in range(4):
        for J in range(4):
            for ty, tx in itertools.product(range(2), range(2)):
                i, j = 2 * I + ty, 2 * J + tx
                exp.append(i * (i - 1) // 2 + j if (j < i < 6) else np.iinfo(np.uint64).max)
    np.testing.assert_array_equal(got, np.array(exp, np.uint64))


@pytest.mark.parametrize("m,n,rho,diag,map_", [(2, 1000, 16, "strict", "lambda"), (2, 1000, 16, "inclusive", "bb"),
                                               (3, 1000, 8, "strict", "lambda"), (3, 100, 4, "inclusive", "lambda"),
                                               (3, 126, 8, "inclusive", "enum"), (2, 100000, 128, "strict", "lambda")])
def test_host_plan_padded(orc, m, n, rho, diag, map_):
    import paper_1610_07394_b200 as sm
    gran = "tile" if rho >= 32 and m == 2 else "thread"
    plan = sm.smap_plan(m, n, rho, map=map_, diag=diag, granularity=gran, device=sm.DEVICE_NONE)
    q = sm.smap_plan_query(plan)
    inc = diag == "inclusive"
    N = orc.padded_n(n + 2 if (m == 3 and inc) else n) // rho
    assert q["grid_blocks"] == orc.grid_blocks(m, inc, map_, N)
    assert q["useful_elems"] == orc.domain_volume(m, inc, n) == sm.smap_volume(m, n, diag)
    assert q["launched_threads"] == q["grid_blocks"] * rho ** m
    # canonical positions
    rng = np.random.default_rng(n)
    for _ in range(50):
        if m == 2:
            i = int(rng.integers(1 if not inc else 0, n))
            j = int(rng.integers(0, i + (1 if inc else 0)))
            assert sm.smap_locate(plan, i, j) == (0, orc.rank2_incl(i, j) if inc else orc.rank2_strict(i, j))
        else:
            t = sorted(int(v) for v in rng.integers(0, n, 3))
            if inc:
                assert sm.smap_locate(plan, *t) == (0, orc.rank3_incl(*t))
            elif t[0] < t[1] < t[2]:
                assert sm.smap_locate(plan, *t) == (0, orc.rank3(*t))


def test_padded_plan_rules():
    import paper_1610_07394_b200 as sm
    N = sm.DEVICE_NONE
    with pytest.raises(Exception):      # sharding a padded grid
        sm.smap_plan(2, 1000, 16, shard_count=2, shard_rank=0, device=N)
    with pytest.raises(Exception):      # tile-blocked layout on a padded grid
        sm.smap_plan(2, 1000, 64, granularity="tile", layout="tiles", device=N)
    with pytest.raises(Exception):      # n below m
        sm.smap_plan(3, 2, 1, device=N)
    with pytest.raises(Exception):      # rho above n'
        sm.smap_plan(2, 5, 16, map="bb", device=N)
    with pytest.raises(Exception):      # lambda3 needs N = n'/rho >= 8
        sm.smap_plan(3, 100, 32, granularity="tile", device=N)
    sm.smap_plan(2, 1000, 16, shard_count=1, device=N)
    sm.smap_plan(2, 1024, 16, shard_count=2, shard_rank=1, device=N)
