"""Oracle pins for the element-level covers (rho^m-thread blocks, P:363-367,
P:383-386; readings E6, E14), the BB baseline, the
launch-order thread dump and the omega_x sharding claims.
CPU only."""
import math

import numpy as np
import pytest

M2 = [(8, 2), (16, 2), (16, 4), (64, 8), (64, 16), (128, 4), (256, 16), (512, 32), (1024, 16)]
M3 = [(16, 2), (32, 2), (32, 4), (64, 4), (64, 8), (128, 8), (128, 16)]


@pytest.mark.parametrize("n,rho", M2)
@pytest.mark.parametrize("inclusive", [False, True])
@pytest.mark.parametrize("bb", [False, True])
def test_cover2_exact(orc, n, rho, inclusive, bb):
    hits, r = orc.element_hits(2, inclusive, bb, n, rho)
    V = n * (n + 1) // 2 if inclusive else n * (n - 1) // 2
    assert len(hits) == V and bool((hits == 1).all())
    assert r["useful"] == V and r["outside"] == 0
    if bb:
        assert r["launched"] == n * n
    elif inclusive:
        assert r["launched"] == n * (n + rho) // 2
        assert r["launched"] - V == n * (rho - 1) // 2          # <= n rho^2
    else:
        assert r["launched"] == n * n // 2
        assert r["launched"] - V == n // 2


@pytest.mark.parametrize("n,rho", M3)
@pytest.mark.parametrize("bb", [False, True])
def test_cover3_exact(orc, n, rho, bb):
    hits, r = orc.element_hits(3, False, bb, n, rho)
    V = math.comb(n, 3)
    assert len(hits) == V and bool((hits == 1).all())
    assert r["useful"] == V and r["outside"] == 0
    if bb:
        assert r["launched"] == n ** 3
    else:
        assert r["launched"] == 3 * n ** 3 // 16
        N = n // rho
        wasted = (rho ** 3 * (3 * N ** 3 // 16 - (N ** 3 - N) // 6 - N)
                  + rho ** 2 * math.comb(N, 2) + N * (rho ** 3 - math.comb(rho, 3)))
        assert r["launched"] - V == wasted


def test_bb_over_lambda_launch_ratio(orc):
    # BB / lambda launched threads: exactly 2 (m=2) and 16/3 (m=3)
    assert orc.element_hits(2, False, True, 256, 16)[1]["launched"] == 2 * orc.element_hits(2, False, False, 256, 16)[1]["launched"]
    a = orc.element_hits(3, False, True, 64, 8)[1]["launched"]
    b = orc.element_hits(3, False, False, 64, 8)[1]["launched"]
    assert 3 * a == 16 * b


def test_thread_dump_matches_hits(orc):
    for m, inc, bb, n, rho in [(2, 0, 0, 64, 8), (2, 1, 0, 64, 8), (2, 0, 1, 32, 4), (3, 0, 0, 64, 4), (3, 0, 1, 32, 4)]:
        d = orc.thread_dump(m, inc, bb, n, rho)
        used = d[d != np.iinfo(np.uint64).max]
        V = orc.domain_volume(m, inc, n)
        assert len(used) == V
        assert np.array_equal(np.sort(used), np.arange(V, dtype=np.uint64))


def test_thread_dump_examples(orc):
    # lambda2 strict, n=16, rho=4 (N=4): block bid=0 is row-0 (w_x=0): diagonal pair D1=0, D2=3
    d = orc.thread_dump(2, 0, 0, 16, 4).reshape(-1, 16)
    MAX = np.iinfo(np.uint64).max
    blk = d[0].reshape(4, 4)            # [ty][tx]
    for ty in range(4):
        for tx in range(4):
            if tx < ty:
                assert blk[ty, tx] == orc.rank2_strict(ty, tx)              # D1 = 0
            elif tx > ty:
                i, j = 12 + 3 - ty, 12 + 3 - tx                              # D2 = 3, reflected
                assert blk[ty, tx] == orc.rank2_strict(i, j)
            else:
                assert blk[ty, tx] == MAX


@pytest.mark.parametrize("m,inc,n,rho", [(2, 0, 1024, 16), (2, 1, 256, 8), (3, 0, 256, 8), (3, 0, 128, 4)])
def test_columns_carry_equal_work(orc, m, inc, n, rho):
    N = n // rho
    w = {orc.column_work(m, inc, n, rho, wx) for wx in range(N // 2)}
    assert len(w) == 1
    V = orc.domain_volume(m, inc, n)
    assert w.pop() * (N // 2) == V


@pytest.mark.parametrize("m,inc,n,rho", [(2, 0, 256, 8), (2, 1, 128, 8), (3, 0, 128, 8)])
@pytest.mark.parametrize("G", [2, 4, 8])
def test_shards_union_is_exact_cover(orc, m, inc, n, rho, G):
    hits = None
    useful = []
    for r in range(G):
        hits, res = orc.element_hits(m, inc, False, n, rho, rank=r, G=G, hits=hits)
        useful.append(res["useful"])
    assert bool((hits == 1).all())
    # every shard carries exactly the same useful volume (section 8e)
    assert len(set(useful)) == 1
