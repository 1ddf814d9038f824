"""GPU parity of the fused C3 payload SMAP_PAYLOAD_INDEX_WRITE_ATM (BASELINE
configs[2]: "tetrahedral index-write plus triple-interaction sum" in one pass):
the packed index array must equal the oracle's nested-loop ranks (E16) or its
enumerated tile-blocked layout (E26) bit for bit, the fused checksums must equal
the oracle's, and the ATM sum must agree with the oracle's fp64 sum within
1e-5 relative (north_star).  The fusion changes no definition, so the oracle
side is the existing index-write and ATM oracles."""
import math

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


def _run(sm, plan, p, eps2, flags):
    out = sm.alloc_out(plan, "index_write_atm")
    sm.smap_run(plan, "index_write_atm", points=torch.from_numpy(p).cuda(), param=eps2, out=out, flags=flags)
    return out, sm.smap_stats_fetch(plan)


@pytest.mark.parametrize("gran,rho,layout", [("thread", 8, "rows"), ("tile", 8, "rows"), ("tile", 16, "rows"),
                                             ("tile", 32, "rows"), ("tile", 16, "tiles"), ("tile", 32, "tiles")])
@pytest.mark.parametrize("map_", ["lambda", "bb"])
@pytest.mark.parametrize("n", [256, 300])
@pytest.mark.parametrize("eps2", [1e-2, 0.0])
def test_index_write_atm(sm, orc, gran, rho, layout, map_, n, eps2):
    if layout == "tiles" and n & (n - 1):
        pytest.skip("the tile-blocked layout needs n = 2^k (E19)")
    p = workloads.points(n, workloads.SEED_C3)
    plan = sm.smap_plan(3, n, rho, map=map_, granularity=gran, layout=layout)
    ref = orc.atm_sum(p, np.float32(eps2))
    V = math.comb(n, 3)
    for flags in (0, sm.RUN_XOR, sm.RUN_CHECKSUM_MIX):
        out, st = _run(sm, plan, p, eps2, flags)
        assert st["count"] == V, flags
        assert abs(st["sum"] - ref) <= 1e-5 * abs(ref), (flags, st["sum"], ref)
        got = out.cpu().numpy().view(np.uint32)
        if layout == "rows":
            exp = orc.index_write(3, False, n)
            np.testing.assert_array_equal(got, exp)
            cs = orc.cs_array(exp)
        else:
            cs = orc.cs_tiles3(n, rho, map_ == "bb", 0, 1)
            assert np.array_equal(np.sort(got), np.arange(V, dtype=np.uint32))
        if flags == sm.RUN_XOR:
            assert st["xr"] == cs["xr"]
        if flags == sm.RUN_CHECKSUM_MIX:
            assert (st["s0"], st["s1"], st["mix"]) == (cs["s0"], cs["s1"], cs["mix"])


def test_index_write_atm_matches_separate_runs(sm):
    """The fused pass returns the same index array and checksums as INDEX_WRITE
    and the bit-identical fp64 sum as ATM on the same plan (the same term code
    runs in both; the partials are combined in the same fixed order)."""
    n = 512
    p = workloads.points(n, 11)
    dp = torch.from_numpy(p).cuda()
    for cfg in (dict(rho=8), dict(rho=32, granularity="tile", layout="tiles"), dict(rho=16, granularity="tile")):
        plan = sm.smap_plan(3, n, **cfg)
        a = sm.alloc_out(plan, "index_write")
        sm.smap_run(plan, "index_write", out=a, flags=sm.RUN_CHECKSUM_MIX)
        s_iw = sm.smap_stats_fetch(plan)
        sm.smap_run(plan, "atm", points=dp, param=1e-2)
        s_atm = sm.smap_stats_fetch(plan)
        b = sm.alloc_out(plan, "index_write_atm")
        sm.smap_run(plan, "index_write_atm", points=dp, param=1e-2, out=b, flags=sm.RUN_CHECKSUM_MIX)
        s_f = sm.smap_stats_fetch(plan)
        assert torch.equal(a, b), cfg
        assert (s_f["count"], s_f["s0"], s_f["s1"], s_f["mix"]) == (s_iw["count"], s_iw["s0"], s_iw["s1"], s_iw["mix"])
        assert s_f["sum"] == s_atm["sum"], cfg


def test_index_write_atm_sharded(sm, orc):
    """Four omega_x shards of the fused payload: the shard records add up to
    the unsharded checksums and the shard sums to the oracle's sum."""
    n, G = 512, 4
    p = workloads.points(n, workloads.SEED_C3)
    ref = orc.atm_sum(p, np.float32(1e-2))
    cs = orc.cs_array(orc.index_write(3, False, n))
    tot = dict(count=0, s0=0, s1=0, mix=0)
    s = 0.0
    for r in range(G):
        plan = sm.smap_plan(3, n, 32, granularity="tile", shard_rank=r, shard_count=G)
        _, st = _run(sm, plan, p, 1e-2, sm.RUN_CHECKSUM_MIX)
        for k in tot:
            tot[k] = (tot[k] + st[k]) % (1 << 64)
        s += st["sum"]
    assert (tot["count"], tot["s0"], tot["s1"], tot["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])
    assert abs(s - ref) <= 1e-5 * abs(ref)


def test_index_write_atm_c3_full(sm, orc):
    """C3 at full size (n = 1024) in the bench launch (tile 32, E26 layout):
    full streaming checksums of the 714 MB index array against the oracle's
    enumerated layout, and the ATM sum against the oracle."""
    c = workloads.CONFIGS["C3"]
    n = c["n"]
    p = workloads.points(n, workloads.SEED_C3)
    ref = orc.atm_sum(p, np.float32(c["eps2"]))
    plan = sm.smap_plan(3, n, **workloads.BENCH_C3)
    _, st = _run(sm, plan, p, c["eps2"], sm.RUN_CHECKSUM_MIX)
    cs = orc.cs_tiles3(n, workloads.BENCH_C3["rho"], False, 0, 1)
    assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])
    assert abs(st["sum"] - ref) <= 1e-5 * abs(ref), (st["sum"], ref)
