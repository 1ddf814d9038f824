"""GPU checks against evaluations that share nothing with the oracle's C code
(VERDICT r01, weak #1 and #2):

* the lambda2 level-square launch order (reading E22) covers every element
  exactly once on the device (hit counts), unsharded and across omega_x shards;
* the fp32 EDM of every product launch, compared element by element with an
  fp64 numpy evaluation of the plain definition ||x_i - x_j||_2 (no fused
  multiply-add, no fp32 rounding) at the north_star's 1e-5 relative bar.  The
  kernel's fp32 result differs from the exact distance by a few ulp (2^-23
  relative each), so the observed maximum is also asserted to stay below 1e-6.
"""
import numpy as np
import pytest

import workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sm():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1610_07394_b200 as s
    return s


@pytest.mark.parametrize("gran,n,rho,G", [("thread", 1024, 16, 1), ("thread", 256, 4, 4), ("thread", 64, 1, 2),
                                          ("tile", 4096, 64, 1), ("tile", 8192, 128, 4), ("thread", 512, 8, 8)])
@pytest.mark.parametrize("diag", ["strict", "inclusive"])
def test_hitcount_square_order(sm, gran, n, rho, G, diag):
    hits = None
    for r in range(G):
        plan = sm.smap_plan(2, n, rho, diag=diag, granularity=gran, order="squares", shard_rank=r, shard_count=G)
        if hits is None:
            hits = sm.alloc_out(plan, "hitcount", zero=True)
        sm.smap_run(plan, "hitcount", out=hits)
    h = hits.cpu().numpy()
    assert len(h) == sm.smap_volume(2, n, diag)
    assert (h == 1).all(), f"missing {(h == 0).sum()} duplicated {(h > 1).sum()}"


def edm_fp64(p):
    """Plain definition in fp64: d[p(i, j)] = sqrt(sum_c (x_jc - x_ic)^2), rows i, j < i."""
    q = p.astype(np.float64)
    n = len(q)
    out = np.empty(n * (n - 1) // 2, np.float64)
    for i in range(1, n):
        d = q[:i] - q[i]
        out[i * (i - 1) // 2:i * (i + 1) // 2] = np.sqrt((d * d).sum(axis=1))
    return out


def canonical(sm, orc, plan_kw, out, n):
    """The device output in canonical packed order (the tile layouts permuted by the oracle's layout map)."""
    got = out.cpu().numpy().view(np.float32)
    if plan_kw.get("layout") != "tiles":
        return got
    pos = orc.tile_layout2(n, plan_kw["rho"], bb=plan_kw.get("map") == "bb")
    return got[pos]


@pytest.mark.parametrize("kw", workloads.BENCH_EDM_VARIANTS, ids=lambda k: "-".join(str(v) for v in k.values()))
@pytest.mark.parametrize("pts", ["uniform", "duplicates", "clustered_scale"])
def test_edm_vs_fp64_definition(sm, orc, kw, pts):
    n = 2048
    if pts == "uniform":
        p = workloads.points(n, workloads.SEED_C2)
    elif pts == "duplicates":
        p = workloads.clustered_points(n, 5)
    else:                                                     # a tight cloud far from the origin
        p = (np.float32(1000.0) + workloads.points(n, 12) * np.float32(1e-2)).astype(np.float32)
    plan = sm.smap_plan(2, n, **kw)
    out = sm.alloc_out(plan, "edm")
    sm.smap_run(plan, "edm", points=torch.from_numpy(p).cuda(), out=out, flags=sm.RUN_XOR)
    got = canonical(sm, orc, kw, out, n).astype(np.float64)
    ref = edm_fp64(p)
    zero = ref == 0.0
    assert (got[zero] == 0.0).all()
    # fp32 differences of fp32 inputs are exact up to one rounding, so the bar is relative to the distance
    rel = np.abs(got[~zero] - ref[~zero]) / ref[~zero]
    assert rel.max() <= 1e-5, rel.max()
    assert rel.max() <= 1e-6, rel.max()


FAST_KW = [dict(rho=256, granularity="tile", map="lambda", layout="tiles"),
           dict(rho=128, granularity="tile", map="lambda", layout="tiles"),
           dict(rho=256, granularity="tile", map="bb", layout="tiles")]


@pytest.mark.parametrize("kw", FAST_KW, ids=lambda k: "-".join(str(v) for v in k.values()))
@pytest.mark.parametrize("pts", ["uniform", "duplicates", "clustered_scale", "tiny"])
def test_edm_fast_sqrt_vs_fp64_definition(sm, orc, kw, pts):
    """SMAP_RUN_FAST_SQRT (sqrt.approx on the vector tile path): every distance within the
    north_star's 1e-5 of the fp64 definition; zero distances exact; a point set with
    coordinates below 2^-40 takes the exact path (bit-identical to the default run)."""
    n = 2048
    if pts == "uniform":
        p = workloads.points(n, workloads.SEED_C2)
    elif pts == "duplicates":
        p = workloads.clustered_points(n, 5)
    elif pts == "clustered_scale":
        p = (np.float32(1000.0) + workloads.points(n, 12) * np.float32(1e-2)).astype(np.float32)
    else:
        # coordinates ~1e-15 (below the 2^-40 staging bound, so every warp must take the
        # exact path) whose squared distances ~1e-30 are still normal fp32 numbers
        p = (workloads.points(n, 13) * np.float32(1e-15)).astype(np.float32)
    plan = sm.smap_plan(2, n, **kw)
    pt = torch.from_numpy(p).cuda()
    fast = sm.alloc_out(plan, "edm")
    exact = sm.alloc_out(plan, "edm")
    sm.smap_run(plan, "edm", points=pt, out=fast, flags=sm.RUN_XOR | sm.RUN_FAST_SQRT)
    assert sm.smap_stats_fetch(plan)["count"] == sm.smap_volume(2, n)
    sm.smap_run(plan, "edm", points=pt, out=exact, flags=sm.RUN_XOR)
    got = canonical(sm, orc, kw, fast, n).astype(np.float64)
    ref = edm_fp64(p)
    zero = ref == 0.0
    assert (got[zero] == 0.0).all()
    rel = np.abs(got[~zero] - ref[~zero]) / ref[~zero]
    assert rel.max() <= 1e-5, rel.max()
    same = torch.equal(fast, exact)
    if pts == "tiny":
        assert same                                            # the staging check sent every warp to the exact path
    elif pts == "uniform":
        assert not same                                        # the approximate path ran (it rounds differently somewhere)


def test_fast_sqrt_flag_is_edm_only(sm):
    plan = sm.smap_plan(2, 1024, 128, granularity="tile", layout="tiles")
    out = sm.alloc_out(plan, "index_write")
    with pytest.raises(sm.SmapError):
        sm.smap_run(plan, "index_write", out=out, flags=sm.RUN_FAST_SQRT)
