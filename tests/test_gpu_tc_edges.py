"""TC edge cases for the pair-bitmap pre-pass (the predicate is
the sign bit of r^2 - R^2, shifted in per row; rows by a warp bit transpose;
32 x 64-blocked bitmap) and the full-adder count: exact ties r^2 == R^2 (must
not count: the paper's triple correlation compares distances < R, and
the oracle compares r^2 < R*R in fp32), R^2 = inf (every triple), R = 0 and
NaN (none), duplicate points (r^2 = 0), at padded n, T = 32 / 64, every TC CTA
size, sharded.  Expected values are the oracle's own brute-force counts."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sm():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1610_07394_b200 as s
    return s


def lattice_points(n, seed):
    """Points of the 8 x 8 x 8 lattice {0, 1/8, ..., 7/8}^3 (exact in fp32, so
    r^2 = (a^2 + b^2 + c^2) / 64 exactly and R = 0.5 gives exact ties), seeded
    order, repeated past 512 points (duplicates: r^2 = 0)."""
    g = np.stack(np.meshgrid(*(np.arange(8),) * 3, indexing="ij"), -1).reshape(-1, 3) / 8.0
    idx = np.random.default_rng(seed).permutation(np.resize(np.arange(512), n))
    return np.ascontiguousarray(g[idx].astype(np.float32))


def tc(sm, n, pts, R, rho, persistent, G=1):
    d = torch.from_numpy(pts).cuda()
    tot = cnt = 0
    for r in range(G):
        plan = sm.smap_plan(3, n, rho, granularity="tile", persistent=persistent, shard_rank=r, shard_count=G)
        sm.smap_run(plan, "tc", points=d, param=R)
        st = sm.smap_stats_fetch(plan)
        tot += st["tc"]
        cnt += st["count"]
    assert cnt == math.comb(n, 3)
    return tot


@pytest.mark.parametrize("R", [0.5, 0.25, 0.375, 1e30, 0.0, float("nan")])
@pytest.mark.parametrize("rho,persistent", [(64, 0), (64, 32), (64, 256), (32, 0)])
def test_tc_ties_and_extreme_thresholds(sm, orc, R, rho, persistent):
    n = 700
    p = lattice_points(n, 41)
    want = orc.tc_count(p, np.float32(R))
    if R == 1e30:
        assert want == math.comb(n, 3)           # (R^2 overflows to inf: every pair is < R^2)
    if R == 0.0 or R != R:
        assert want == 0
    assert tc(sm, n, p, np.float32(R), rho, persistent) == want


@pytest.mark.parametrize("G", [2, 4])
def test_tc_ties_sharded(sm, orc, G):
    n = 1024                                      # (shards need power-of-two n and G)
    p = lattice_points(n, 43)
    want = orc.tc_count(p, np.float32(0.5))
    assert tc(sm, n, p, np.float32(0.5), 64, 16, G) == want


# ---- large bitmaps (>= 128 blocks per side: C5X size)
def _golden_c5x():
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "bench_expected.json")) as f:
        return json.load(f)["C5X"]


@pytest.mark.parametrize("G,persistent", [(1, 256), (8, 256), (2, 16)])
def test_c5x_full_size(sm, G, persistent):
    """C5X (n = 8192, the supplementary scaling workload) at full size, unsharded and
    sharded: the shard counts add up to the oracle-written golden count
    (tests/golden/bench_expected.json, scripts/make_bench_golden.py)."""
    import workloads
    g = _golden_c5x()
    p = workloads.points(g["n"], g["seed"])
    assert tc(sm, g["n"], p, np.float32(g["R"]), 64, persistent, G) == g["tc"]


@pytest.mark.parametrize("map_,n", [("lambda", 4100), ("bb", 4096)])
def test_large_bitmap_vs_oracle(sm, orc, map_, n):
    """The pre-pass and the 64-thread count at n > 4096 (a padded n: the last bitmap
    blocks partly outside the point set) and with the BB map, against the oracle's
    brute-force count."""
    import workloads
    p = workloads.points(n, 47)
    d = torch.from_numpy(p).cuda()
    plan = sm.smap_plan(3, n, 64, map=map_, granularity="tile", persistent=32)
    sm.smap_run(plan, "tc", points=d, param=0.5)
    st = sm.smap_stats_fetch(plan)
    assert st["count"] == math.comb(n, 3)
    assert st["tc"] == orc.tc_count(p, np.float32(0.5))
