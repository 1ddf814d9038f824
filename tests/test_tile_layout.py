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
    p3 = sm.smap_plan(3, 64, 8, device=sm.DEVICE_NONE)
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
