"""Oracle pins for the enumeration-map baseline (SMAP_MAP_ENUM):
the linear enumeration g: Z^1 -> Z^m of P:166-174 applied at block level
(P:252-262).  The oracle finds a block by walking the rows (no roots); these
pins check it against itertools enumerations of the block simplices, the
closed-form grid sizes, and exact element covers.  CPU only."""
import itertools
import math

import numpy as np
import pytest


@pytest.mark.parametrize("N", [1, 2, 3, 8, 64])
def test_enum2_block_order_is_row_major_lower_triangle(orc, N):
    d = orc.map_dump(2, False, "enum", N)
    exp = [(J, I) for I in range(N) for J in range(I + 1)]           # row-major {J <= I}
    assert len(d) == N * (N + 1) // 2 == orc.grid_blocks(2, False, "enum", N)
    assert [tuple(r[:2]) for r in d.tolist()] == exp
    assert all(r[3] == (0 if r[0] < r[1] else 3) for r in d.tolist())


@pytest.mark.parametrize("N", [1, 2, 5, 16])
def test_enum3_block_order_is_colex_tetrahedron(orc, N):
    d = orc.map_dump(3, False, "enum", N)
    # colex order of multisets I <= J <= K: K outermost, I innermost
    exp = [(I, J, K) for K in range(N) for J in range(K + 1) for I in range(J + 1)]
    assert len(d) == math.comb(N + 2, 3) == orc.grid_blocks(3, False, "enum", N)
    assert [tuple(r[:3]) for r in d.tolist()] == exp
    for I, J, K, c in d.tolist():
        want = 0 if I < J < K else 5 if I == J < K else 6 if I < J == K else 2
        assert c == want


@pytest.mark.parametrize("m,inclusive,n,rho", [(2, False, 64, 4), (2, True, 64, 4), (2, False, 256, 16),
                                               (3, False, 32, 2), (3, False, 64, 4)])
def test_enum_element_cover_exact(orc, m, inclusive, n, rho):
    hits, r = orc.element_hits(m, inclusive, "enum", n, rho)
    assert (hits == 1).all() and r["outside"] == 0
    N = n // rho
    nb = N * (N + 1) // 2 if m == 2 else math.comb(N + 2, 3)
    assert r["launched"] == nb * rho ** m
    V = orc.domain_volume(m, inclusive, n)
    assert r["useful"] == V
    # waste: m=2 strict n(rho+1)/2, inclusive n(rho-1)/2 -- the diagonal blocks' upper halves
    if m == 2:
        assert r["launched"] - V == (n * (rho - 1) // 2 if inclusive else n * (rho + 1) // 2)


def test_enum_thread_dump_matches_brute_force(orc):
    # every launched thread of the ENUM grid: block from the enumeration, element = identity + filter
    n, rho = 32, 4
    N = n // rho
    got = orc.thread_dump(2, False, "enum", n, rho)
    exp = []
    for I in range(N):
        for J in range(I + 1):
            for ty, tx in itertools.product(range(rho), range(rho)):
                i, j = I * rho + ty, J * rho + tx
                exp.append(i * (i - 1) // 2 + j if j < i else np.iinfo(np.uint64).max)
    np.testing.assert_array_equal(got, np.array(exp, np.uint64))


@pytest.mark.parametrize("m,n,rho,diag", [(2, 1024, 16, "strict"), (2, 1024, 16, "inclusive"), (3, 1024, 8, "strict")])
def test_enum_host_plan_closed_forms(orc, m, n, rho, diag):
    """The C library's host-only plan (no device) reports the enumeration grid
    and its waste in closed form, equal to the oracle's walk."""
    import paper_1610_07394_b200 as sm
    plan = sm.smap_plan(m, n, rho, map="enum", diag=diag, device=sm.DEVICE_NONE)
    q = sm.smap_plan_query(plan)
    N = n // rho
    assert q["grid_blocks"] == orc.grid_blocks(m, diag == "inclusive", "enum", N)
    assert q["launched_threads"] == q["grid_blocks"] * rho ** m
    assert q["useful_elems"] == sm.smap_volume(m, n, diag)
    assert q["wasted_threads"] == q["launched_threads"] - q["useful_elems"]
    with pytest.raises(Exception):
        sm.smap_plan(m, n, rho, map="enum", diag=diag, granularity="tile", device=sm.DEVICE_NONE)
    with pytest.raises(Exception):
        sm.smap_plan(m, n, rho, map="enum", diag=diag, shard_count=2, shard_rank=1, device=sm.DEVICE_NONE)
