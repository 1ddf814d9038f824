"""Any n by "approach n from below" (reading E28):
the M tiles per side are cut into the binary digits of M and every piece is a
power-of-two simplex mapped by lambda or a box at the identity.  Oracle pins
(CPU): the segments are the binary digits; the tile records cover the tile
domain exactly once with no launched tile outside it (m=2) or only lambda3's
own idle tiles (m=3, closed form); a power-of-two M reduces to the plain
lambda2 / lambda3 tile grid; element covers against the nested-loop domains
for non-power-of-two n; the C library's host-only plans report the same tile
counts."""
import itertools
import math

import numpy as np
import pytest


@pytest.mark.parametrize("M", list(range(1, 200)) + [1023, 1024, 1025, 4095, 65537])
def test_segments_are_binary_digits(orc, M):
    Ns, Os = orc.below_segments(M)
    assert sum(Ns) == M
    assert Ns == sorted(Ns, reverse=True) and len(set(Ns)) == len(Ns)
    assert all(x & (x - 1) == 0 for x in Ns)
    assert Ns == [1 << b for b in range(M.bit_length()) if M >> b & 1][::-1]
    assert Os == [sum(Ns[:s]) for s in range(len(Ns))]


@pytest.mark.parametrize("M", list(range(1, 70)) + [127, 200, 333])
def test_m2_tiles_cover_exactly_without_waste(orc, M):
    rec = orc.below_tiles(2, M)
    assert len(rec) == M * (M + 1) // 2                 # every launched tile is in the domain
    pairs = [(int(J), int(I)) for J, I, _, _ in rec]
    assert len(set(pairs)) == len(pairs)
    assert set(pairs) == {(J, I) for I in range(M) for J in range(I + 1)}
    assert all((c == 2) == (J == I) for J, I, _, c in rec)
    assert (rec[:, 2] == 0).all()


def _lambda3_idle(N):
    # lambda3 grid (N/2, N/2, 3N/4) minus the (N^3 - N)/6 tiles I <= J < K and the N body tiles
    return 3 * N ** 3 // 16 - (N ** 3 - N) // 6 - N


@pytest.mark.parametrize("M", list(range(1, 40)) + [64, 100, 129])
def test_m3_tiles_cover_exactly(orc, M):
    rec = orc.below_tiles(3, M)
    bb = []                                            # BB tiles I <= J <= K each record carries
    idle = 0
    for I, J, K, c in (tuple(int(v) for v in r) for r in rec):
        if c == 3:
            idle += 1
            assert I == J == K == 0
        elif c == 2:
            assert I == J == K
            bb.append((I, I, I))
        elif c in (0, 1) and I == J:                   # lambda3 face tile: both folded sets (E14)
            assert J < K
            bb += [(I, I, K), (I, K, K)]
        elif c == 5:
            assert I == J < K
            bb.append((I, J, K))
        elif c == 6:
            assert I < J == K
            bb.append((I, J, K))
        else:
            assert c in (0, 1) and I < J < K
            bb.append((I, J, K))
    assert len(set(bb)) == len(bb) == math.comb(M + 2, 3)
    assert set(bb) == set(itertools.combinations_with_replacement(range(M), 3))
    Ns, _ = orc.below_segments(M)
    assert idle == sum(_lambda3_idle(N) for N in Ns if N >= 8)


@pytest.mark.parametrize("M", [2, 4, 8, 16, 64, 256])
def test_m2_power_of_two_is_the_lambda2_grid(orc, M):
    """One segment: the decomposition is the lambda2 inclusive tile grid itself."""
    np.testing.assert_array_equal(orc.below_tiles(2, M), orc.map_dump(2, True, False, M))


@pytest.mark.parametrize("M", [8, 16, 32, 64])
def test_m3_power_of_two_is_the_lambda3_grid(orc, M):
    np.testing.assert_array_equal(orc.below_tiles(3, M), orc.map_dump(3, False, False, M))


@pytest.mark.parametrize("m,inc,n,T", [(2, False, 1000, 32), (2, True, 1000, 32), (2, False, 333, 8), (2, True, 70, 4),
                                       (2, False, 2, 1), (2, True, 1, 1), (2, False, 97, 1),
                                       (3, False, 100, 8), (3, True, 100, 8), (3, False, 37, 4), (3, True, 37, 4),
                                       (3, False, 300, 16), (3, False, 3, 1), (3, False, 45, 1), (3, True, 1, 1)])
def test_element_cover_exact(orc, m, inc, n, T):
    hits, r = orc.below_element_hits(m, inc, n, T)
    assert len(hits) == orc.domain_volume(m, inc, n)
    assert (hits == 1).all() and r["outside"] == 0 and r["useful"] == len(hits)


def test_element_cover_detects_a_corrupted_tile(orc):
    """The cover check is not vacuous: dropping or duplicating one record of
    the tile list breaks it (checked on the plain record list)."""
    M, T = 5, 2
    rec = orc.below_tiles(2, M)
    cover = {}
    for J, I, _, c in rec[1:]:                         # drop the first record
        for r in range(T):
            for cc in range(T):
                if c == 2 and cc >= r:
                    continue
                key = (I * T + r, J * T + cc)
                cover[key] = cover.get(key, 0) + 1
    assert len(cover) < math.comb(M * T, 2)


@pytest.mark.parametrize("m,n,T", [(2, 1000, 32), (2, 65535, 256), (2, 100000, 128), (3, 1000, 32), (3, 1500, 8),
                                   (3, 2047, 64)])
@pytest.mark.parametrize("diag", ["strict", "inclusive"])
def test_host_plan_counts(orc, m, n, T, diag):
    import paper_1610_07394_b200 as sm
    plan = sm.smap_plan(m, n, T, map="below", diag=diag, granularity="tile", device=sm.DEVICE_NONE)
    q = sm.smap_plan_query(plan)
    nint = n + 2 if (m == 3 and diag == "inclusive") else n
    M = -(-nint // T)
    assert q["grid_blocks"] == len(orc.below_tiles(m, M))
    assert q["launched_threads"] == q["grid_blocks"] * T ** m
    assert q["useful_elems"] == orc.domain_volume(m, diag == "inclusive", n)


def test_host_plan_rejects(orc):
    import paper_1610_07394_b200 as sm
    N = sm.DEVICE_NONE
    with pytest.raises(sm.SmapError):                                        # THREAD + tile layout
        sm.smap_plan(2, 1000, 16, map="below", layout="tiles", device=N)
    with pytest.raises(sm.SmapError):
        sm.smap_plan(2, 1000, 32, map="below", granularity="tile", shard_count=2, device=N)
    with pytest.raises(sm.SmapError):                                        # lambda m=3 inclusive tile layout
        sm.smap_plan(3, 1022, 32, map="lambda", diag="inclusive", granularity="tile", layout="tiles", device=N)


@pytest.mark.parametrize("m,inc,n,T", [(2, False, 100, 8), (2, True, 37, 4), (2, False, 64, 8), (2, False, 1000, 32),
                                       (3, False, 100, 8), (3, False, 64, 8), (3, False, 37, 4), (3, True, 37, 4),
                                       (3, False, 130, 16)])
def test_tile_layout_e29(orc, m, inc, n, T):
    """E29: every rank gets one position, positions are distinct, tiles are
    contiguous slots in launch order, and the holes are exactly the elements
    cut by n (none when T divides n')."""
    pos, L = orc.below_tile_layout(m, inc, n, T)
    V = orc.domain_volume(m, inc, n)
    assert len(pos) == V and (pos >= 0).all() and len(np.unique(pos)) == V and pos.max() < L
    nint = n + 2 if (m == 3 and inc) else n
    if nint % T == 0:
        assert L == V
    else:
        assert L > V
    # the streaming checksum walks the same layout
    cs = orc.cs_below_tiles("index_write", m, inc, n, T)
    M = 1 << 64
    assert cs["count"] == V
    assert cs["s1"] == int(sum((int(p) + 1) * r for r, p in enumerate(pos)) % M)


@pytest.mark.parametrize("m,n,T", [(2, 1000, 32), (2, 70000, 128), (3, 1100, 32), (3, 300, 8)])
@pytest.mark.parametrize("diag", ["strict", "inclusive"])
def test_host_plan_tile_layout_bytes(orc, m, n, T, diag):
    import paper_1610_07394_b200 as sm
    plan = sm.smap_plan(m, n, T, map="below", diag=diag, granularity="tile", layout="tiles", device=sm.DEVICE_NONE)
    V = orc.domain_volume(m, diag == "inclusive", n)
    if n <= 1100 and (m == 2 or n <= 300):
        _, L = orc.below_tile_layout(m, diag == "inclusive", n, T)
    else:                                   # closed form: full tiles T^m plus the class-sized diagonal slots
        L = None
    nb = sm.smap_out_bytes(plan, "index_write")
    elem = 8 if V > (1 << 32) else 4
    if L is not None:
        assert nb == L * elem
    assert nb >= V * elem
    if L is not None and V <= 600000:                  # smap_locate inverts E29 (host): every element
        pos, _ = orc.below_tile_layout(m, diag == "inclusive", n, T)
        got = _locate_all(sm, plan, m, n, diag == "inclusive")
        np.testing.assert_array_equal(got, pos)


def _locate_all(sm, plan, m, n, inc):
    out = []
    if m == 2:
        for i in range(n):
            for j in range(i + 1 if inc else i):
                out.append(sm.smap_locate(plan, i, j)[1])
    else:                                   # nested-loop (packed rank) order
        for k in range(n):
            for j in range(k + 1 if inc else k):
                for i in range(j + 1 if inc else j):
                    out.append(sm.smap_locate(plan, i, j, k)[1])
    return np.array(out, np.int64)


@pytest.mark.parametrize("m,inc,n,T", [(2, False, 333, 32), (2, True, 700, 64), (2, False, 130, 32), (2, True, 1000, 32),
                                       (3, False, 100, 8), (3, False, 130, 16), (3, False, 64, 8), (3, False, 99, 8),
                                       (3, True, 100, 8), (3, True, 62, 8)])
def test_locate_inverts_e29(orc, m, inc, n, T):
    import paper_1610_07394_b200 as sm
    plan = sm.smap_plan(m, n, T, map="below", diag="inclusive" if inc else "strict", granularity="tile",
                        layout="tiles", device=sm.DEVICE_NONE)
    pos, _ = orc.below_tile_layout(m, inc, n, T)
    np.testing.assert_array_equal(_locate_all(sm, plan, m, n, inc), pos)
