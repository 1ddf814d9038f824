"""The lambda-order tile-blocked output layout (E23):
the oracle defines it by enumeration (or_tile_layout2), the C library locates
elements in O(1) (smap_locate), the GPU writes it (-m gpu)."""
import math

import numpy as np
import pytest

import workloads

CASES = [(512, 32, False, False, 1), (512, 32, True, False, 1), (512, 64, False, True, 1), (256, 32, True, True, 1),
         (1024, 64, False, False, 4), (256, 32, True, False, 2), (2048, 128, False, False, 8)]


def _unrank2(p, inclusive):
    """(i, j) of canonical packed rank p (plain search)."""
    i = int((math.isqrt(8 * p + 1) + (-1 if inclusive else 1)) // 2)
    base = (lambda i: i * (i + 1) // 2) if inclusive else (lambda i: i * (i - 1) // 2)
    while base(i) > p:
        i -= 1
    while base(i + 1) <= p:
        i += 1
    return i, p - base(i)


@pytest.mark.parametrize("n,T,inc,bb,G", CASES)
def test_layout_is_a_partition_and_locate_agrees(orc, n, T, inc, bb, G):
    import paper_1610_07394_b200 as sm
    diag = "inclusive" if inc else "strict"
    V = orc.domain_volume(2, inc, n)
    owner = np.full(V, -1, np.int64)
    rng = np.random.default_rng(n + T)
    for r in range(G):
        pos = orc.tile_layout2(n, T, inc, bb, r, G)
        own = np.nonzero(pos >= 0)[0]
        assert np.array_equal(np.sort(pos[own]), np.arange(len(own)))      # bijection onto [0, V/G)
        assert (owner[own] == -1).all()
        owner[own] = r
        plan = sm.smap_plan(2, n, T, map="bb" if bb else "lambda", diag=diag, granularity="tile", shard_rank=r,
                            shard_count=G, device=sm.DEVICE_NONE, layout="tiles")
        assert sm.smap_plan_query(plan)["useful_elems"] == len(own) == V // G
        for p in rng.choice(own, size=min(400, len(own)), replace=False):
            i, j = _unrank2(int(p), inc)
            assert sm.smap_locate(plan, i, j) == (r, int(pos[p]))
    assert (owner >= 0).all()


@pytest.mark.parametrize("n,T,inc,bb,G", CASES)
def test_streaming_tile_checksum_equals_materialised(orc, n, T, inc, bb, G):
    p = workloads.points(n, 3)
    iw = orc.index_write(2, inc, n)
    ed = None if inc else orc.edm(p)
    for r in range(G):
        assert orc.cs_tiles2("index_write", n, T, inc, bb, r, G) == orc.cs_array(orc.to_tile_layout2(iw, n, T, inc, bb, r, G))
        if ed is not None:
            assert orc.cs_tiles2("edm", n, T, inc, bb, r, G, points=p) == \
                orc.cs_array(orc.to_tile_layout2(ed, n, T, inc, bb, r, G))


def test_lambda2_inverse_closed_form(orc):
    # the O(1) inverse used by smap_locate: b = 2^floor(log2(I^J)), q = I >> (log2 b + 1)
    for N in (2, 8, 64, 512):
        for wy in range(1, N):
            for wx in range(N // 2):
                J, I = orc.lambda2(wx, wy)
                l = (I ^ J).bit_length() - 1
                q = I >> (l + 1)
                assert (J - q * (1 << l), I - 2 * q * (1 << l)) == (wx, wy)


def test_locate_rows_layout_and_errors():
    import paper_1610_07394_b200 as sm
    plan = sm.smap_plan(2, 1024, 16, shard_count=4, device=sm.DEVICE_NONE)
    sh, pos = sm.smap_locate(plan, 700, 3)
    assert pos == 700 * 699 // 2 + 3 and 0 <= sh < 4
    with pytest.raises(sm.SmapError):
        sm.smap_locate(plan, 3, 700)               # above the diagonal
    p3 = sm.smap_plan(3, 64, 8, device=sm.DEVICE_NONE)          # THREAD, canonical
    assert sm.smap_locate(p3, 1, 5, 9) == (0, math.comb(9, 3) + math.comb(5, 2) + 1)
    with pytest.raises(sm.SmapError):
        sm.smap_plan(2, 1024, 16, layout="tiles", device=sm.DEVICE_NONE)          # THREAD granularity


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("n,T,inc,bb,G", CASES + [(4096, 256, False, False, 2), (2048, 128, False, True, 1)])
def test_gpu_tile_layout_parity(orc, n, T, inc, bb, G):
    torch = pytest.importorskip("torch")
    import paper_1610_07394_b200 as sm
    diag = "inclusive" if inc else "strict"
    p = workloads.points(n, 11)
    dp = torch.from_numpy(p).cuda()
    iw = orc.index_write(2, inc, n)
    ed = orc.edm(p) if not inc else None
    for r in range(G):
        plan = sm.smap_plan(2, n, T, map="bb" if bb else "lambda", diag=diag, granularity="tile", shard_rank=r,
                            shard_count=G, layout="tiles")
        # index write: values are canonical ranks, stored at tile positions
        out = sm.alloc_out(plan, "index_write")
        sm.smap_run(plan, "index_write", out=out, flags=sm.RUN_CHECKSUM_MIX)
        st = sm.smap_stats_fetch(plan)
        exp = orc.to_tile_layout2(iw, n, T, inc, bb, r, G)
        np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), exp)
        cs = orc.cs_array(exp)
        assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])
        # exact cover at tile positions
        h = sm.alloc_out(plan, "hitcount", zero=True)
        sm.smap_run(plan, "hitcount", out=h)
        assert (h.cpu().numpy() == 1).all()
        if ed is not None:
            exp = orc.to_tile_layout2(ed, n, T, inc, bb, r, G)
            cse = orc.cs_array(exp)
            for flags in (0, sm.RUN_XOR, sm.RUN_CHECKSUM, sm.RUN_CHECKSUM_MIX):
                o = sm.alloc_out(plan, "edm")
                sm.smap_run(plan, "edm", points=dp, out=o, flags=flags)
                st = sm.smap_stats_fetch(plan)
                assert np.array_equal(o.cpu().numpy().view(np.uint32), exp.view(np.uint32)), flags
                if flags:
                    assert st["count"] == cse["count"], flags
                if flags == sm.RUN_XOR:
                    assert st["xr"] == cse["xr"]
                if flags & (sm.RUN_CHECKSUM | sm.RUN_CHECKSUM_MIX):
                    assert (st["s0"], st["s1"]) == (cse["s0"], cse["s1"]), flags


# ---------------------------------------------------------------- m=3 (reading E26)
CASES3 = [(64, 8, False, 1), (64, 8, True, 1), (128, 8, False, 4), (128, 16, False, 2), (256, 32, False, 1),
          (256, 16, True, 1), (512, 32, False, 8)]


def _unrank3(p):
    """(i, j, k) of canonical triple rank p (plain search)."""
    k = 2
    while math.comb(k + 1, 3) <= p:
        k += 1
    rem = p - math.comb(k, 3)
    j = 1
    while math.comb(j + 1, 2) <= rem:
        j += 1
    return rem - math.comb(j, 2), j, k


@pytest.mark.parametrize("n,T,bb,G", CASES3)
def test_layout3_partition_and_locate_agrees(orc, n, T, bb, G):
    """The oracle's enumerated E26 layout is a partition of the triples into G
    shard-local arrays of C(n,3)/G slots (lambda: every omega_x column carries
    equal work), and smap_locate's closed-form slots with the lambda3 inverse
    (b = 2^floor(log2(I^K)), q = I >> (log2 b + 1), inside iff Z < b) agree."""
    import paper_1610_07394_b200 as sm
    V = math.comb(n, 3)
    owner = np.full(V, -1, np.int64)
    rng = np.random.default_rng(n + T)
    for r in range(G):
        pos = orc.tile_layout3(n, T, bb, r, G)
        own = np.nonzero(pos >= 0)[0]
        assert np.array_equal(np.sort(pos[own]), np.arange(len(own)))
        assert (owner[own] == -1).all()
        owner[own] = r
        if not bb:
            assert len(own) * G == V
        plan = sm.smap_plan(3, n, T, map="bb" if bb else "lambda", granularity="tile", shard_rank=r,
                            shard_count=G, device=sm.DEVICE_NONE, layout="tiles")
        assert sm.smap_out_bytes(plan, "index_write") == 4 * len(own)
        for p in rng.choice(own, size=min(1500, len(own)), replace=False):
            assert sm.smap_locate(plan, *_unrank3(int(p))) == (r, pos[p])
    assert (owner >= 0).all()


def test_layout3_streaming_checksum(orc):
    n, T = 128, 16
    iw = orc.index_write(3, False, n)
    for bb, G in ((False, 1), (False, 4), (True, 1)):
        for r in range(G):
            exp = orc.to_tile_layout3(iw, n, T, bb, r, G)
            cs = orc.cs_array(exp)
            assert orc.cs_tiles3(n, T, bb, r, G) == cs


@pytest.mark.gpu
@pytest.mark.parametrize("n,T,bb,G", CASES3 + [(1024, 32, False, 2)])
def test_gpu_tile_layout3_parity(orc, n, T, bb, G):
    pytest.importorskip("torch")
    import paper_1610_07394_b200 as sm
    iw = orc.index_write(3, False, n)
    for r in range(G):
        plan = sm.smap_plan(3, n, T, map="bb" if bb else "lambda", granularity="tile", shard_rank=r,
                            shard_count=G, layout="tiles")
        exp = orc.to_tile_layout3(iw, n, T, bb, r, G)
        cs = orc.cs_array(exp)
        for flags in (sm.RUN_CHECKSUM_MIX, sm.RUN_XOR):
            out = sm.alloc_out(plan, "index_write")
            sm.smap_run(plan, "index_write", out=out, flags=flags)
            st = sm.smap_stats_fetch(plan)
            np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), exp)
            if flags == sm.RUN_XOR:
                assert (st["count"], st["xr"]) == (cs["count"], cs["xr"])
            else:
                assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])
        h = sm.alloc_out(plan, "hitcount", zero=True)
        sm.smap_run(plan, "hitcount", out=h)
        assert (h.cpu().numpy() == 1).all()
