"""GPU parity of the approach-from-below map (SMAP_MAP_BELOW; P:399-404,
reading E28) through the C ABI: tile records bit-exact against the oracle's
decomposition, exact element covers, and every payload against the oracle for
non-power-of-two n (bit-exact indices, EDM and counts; ATM sum within 1e-5)."""
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


def run(sm, plan, payload, points=None, param=0.0, flags=0, zero=False):
    out = sm.alloc_out(plan, payload, zero=zero)
    sm.smap_run(plan, payload, points=points, param=param, out=out, flags=flags)
    return out, sm.smap_stats_fetch(plan)


def dev(p):
    return torch.from_numpy(np.ascontiguousarray(p)).cuda()


@pytest.mark.parametrize("m,n,T", [(2, 1000, 32), (2, 5000, 128), (2, 4096, 64), (2, 33, 32), (2, 70000, 512),
                                   (3, 1000, 32), (3, 300, 8), (3, 1024, 16), (3, 9, 8), (3, 700, 64)])
@pytest.mark.parametrize("diag", ["strict", "inclusive"])
def test_map_dump(sm, orc, m, n, T, diag):
    plan = sm.smap_plan(m, n, T, map="below", diag=diag, granularity="tile")
    out, _ = run(sm, plan, "map_dump")
    nint = n + 2 if (m == 3 and diag == "inclusive") else n
    exp = orc.below_tiles(m, -(-nint // T))
    np.testing.assert_array_equal(out.cpu().numpy().reshape(-1, 4), exp)


@pytest.mark.parametrize("m,n,T", [(2, 1000, 32), (2, 3000, 64), (2, 12345, 256), (2, 100, 512), (2, 2, 32),
                                   (3, 1000, 32), (3, 300, 8), (3, 333, 16), (3, 3, 8), (3, 520, 64), (3, 129, 8)])
@pytest.mark.parametrize("diag", ["strict", "inclusive"])
def test_hitcount_exact_cover(sm, m, n, T, diag):
    plan = sm.smap_plan(m, n, T, map="below", diag=diag, granularity="tile")
    out, _ = run(sm, plan, "hitcount", zero=True)
    assert out.numel() == sm.smap_volume(m, n, diag)
    assert bool((out == 1).all()), f"missing {(out == 0).sum().item()} duplicated {(out > 1).sum().item()}"


@pytest.mark.parametrize("m,n,T", [(2, 1500, 32), (2, 1500, 128), (2, 777, 512), (3, 300, 8), (3, 300, 16),
                                   (3, 300, 32), (3, 200, 64)])
@pytest.mark.parametrize("diag", ["strict", "inclusive"])
def test_index_write(sm, orc, m, n, T, diag):
    plan = sm.smap_plan(m, n, T, map="below", diag=diag, granularity="tile")
    out, st = run(sm, plan, "index_write", flags=sm.RUN_CHECKSUM_MIX)
    exp = orc.index_write(m, diag == "inclusive", n)
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), exp)
    cs = orc.cs_array(exp)
    assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])


@pytest.mark.parametrize("n,T", [(1500, 32), (3001, 64), (2900, 128), (5000, 256), (1000, 512)])
def test_edm_bit_exact(sm, orc, n, T):
    p = workloads.points(n, workloads.SEED_C2)
    plan = sm.smap_plan(2, n, T, map="below", granularity="tile")
    exp = orc.edm(p)
    cs = orc.cs_array(exp)
    for flags in (0, sm.RUN_XOR, sm.RUN_CHECKSUM):
        out, st = run(sm, plan, "edm", points=dev(p), flags=flags)
        assert np.array_equal(out.cpu().numpy().view(np.uint32), exp.view(np.uint32)), flags
        if flags == sm.RUN_XOR:
            assert (st["count"], st["xr"]) == (cs["count"], cs["xr"])
        if flags == sm.RUN_CHECKSUM:
            assert (st["count"], st["s0"], st["s1"]) == (cs["count"], cs["s0"], cs["s1"])


@pytest.mark.parametrize("n,T", [(300, 8), (300, 16), (333, 32), (250, 32), (20, 8), (45, 16)])
def test_atm_tc_iwa(sm, orc, n, T):
    p = workloads.points(n, workloads.SEED_C3)
    dp = dev(p)
    plan = sm.smap_plan(3, n, T, map="below", granularity="tile")
    V = math.comb(n, 3)
    ref = orc.atm_sum(p, np.float32(1e-2))
    _, st = run(sm, plan, "atm", points=dp, param=1e-2)
    assert st["count"] == V
    assert abs(st["sum"] - ref) <= 1e-5 * abs(ref), (st["sum"], ref)
    out, st = run(sm, plan, "index_write_atm", points=dp, param=1e-2, flags=sm.RUN_XOR)
    assert st["count"] == V and abs(st["sum"] - ref) <= 1e-5 * abs(ref)
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), np.arange(V, dtype=np.uint32))
    for R in (0.5, 0.2):                                # (M*T need not be a multiple of 32)
        _, st = run(sm, plan, "tc", points=dp, param=R)
        assert st["tc"] == orc.tc_count(p, np.float32(R)) and st["count"] == V


@pytest.mark.parametrize("n", [100, 700, 2100])
def test_tc_tile64(sm, orc, n):
    p = workloads.points(n, workloads.SEED_C5)
    plan = sm.smap_plan(3, n, 64, map="below", granularity="tile", persistent=8)
    _, st = run(sm, plan, "tc", points=dev(p), param=0.5)
    assert st["tc"] == orc.tc_count(p, np.float32(0.5)) and st["count"] == math.comb(n, 3)


def test_below_vs_above_full_size(sm, orc):
    """A non-power-of-two C2-like EDM (n = 40000, 800 M pairs): both ways of
    handling any n give the same checksums as the oracle."""
    n = 40000
    p = workloads.points(n, workloads.SEED_C2)
    cs = orc.cs_edm(p)
    dp = dev(p)
    for mp in ("below", "lambda"):
        plan = sm.smap_plan(2, n, 128, map=mp, granularity="tile")
        out, st = run(sm, plan, "edm", points=dp, flags=sm.RUN_CHECKSUM_MIX)
        assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"]), mp
        del out
        torch.cuda.empty_cache()


SENT = 0x7FABCDEF


@pytest.mark.parametrize("m,n,T", [(2, 1000, 32), (2, 1500, 128), (2, 777, 512), (2, 1024, 64), (3, 300, 8),
                                   (3, 300, 16), (3, 333, 32), (3, 256, 32), (3, 200, 64)])
@pytest.mark.parametrize("diag", ["strict", "inclusive"])
def test_tile_layout_index_write(sm, orc, m, n, T, diag):
    """E29: every packed rank lands at the oracle's position and the holes of
    tiles cut by n are never written."""
    plan = sm.smap_plan(m, n, T, map="below", diag=diag, granularity="tile", layout="tiles")
    pos, L = orc.below_tile_layout(m, diag == "inclusive", n, T)
    out = sm.alloc_out(plan, "index_write")
    assert out.numel() == L
    out.fill_(SENT)
    sm.smap_run(plan, "index_write", out=out, flags=sm.RUN_CHECKSUM_MIX)
    st = sm.smap_stats_fetch(plan)
    got = out.cpu().numpy().view(np.uint32)
    V = len(pos)
    np.testing.assert_array_equal(got[pos], np.arange(V, dtype=np.uint32))
    holes = np.ones(L, bool)
    holes[pos] = False
    assert (got[holes] == SENT).all()
    cs = orc.cs_below_tiles("index_write", m, diag == "inclusive", n, T)
    assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])


@pytest.mark.parametrize("n,T", [(1500, 64), (3001, 128), (5000, 256), (4096, 128)])
def test_tile_layout_edm(sm, orc, n, T):
    p = workloads.points(n, workloads.SEED_C2)
    plan = sm.smap_plan(2, n, T, map="below", granularity="tile", layout="tiles")
    pos, L = orc.below_tile_layout(2, False, n, T)
    exp = orc.edm(p)
    for flags in (0, sm.RUN_XOR, sm.RUN_CHECKSUM):
        out, st = run(sm, plan, "edm", points=dev(p), flags=flags)
        got = out.cpu().numpy().view(np.uint32)
        np.testing.assert_array_equal(got[pos], exp.view(np.uint32))
        if flags:
            cs = orc.cs_below_tiles("edm", 2, False, n, T, points=p)
            assert st["count"] == cs["count"]
            assert (st["xr"] if flags == sm.RUN_XOR else st["s1"]) == (cs["xr"] if flags == sm.RUN_XOR else cs["s1"])


@pytest.mark.parametrize("n,T", [(300, 16), (333, 32), (1100, 32)])
def test_tile_layout_fused_iwa(sm, orc, n, T):
    p = workloads.points(n, workloads.SEED_C3)
    plan = sm.smap_plan(3, n, T, map="below", granularity="tile", layout="tiles")
    out, st = run(sm, plan, "index_write_atm", points=dev(p), param=1e-2, flags=sm.RUN_CHECKSUM_MIX)
    cs = orc.cs_below_tiles("index_write", 3, False, n, T)
    assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])
    ref = orc.atm_sum(p, np.float32(1e-2))
    assert abs(st["sum"] - ref) <= 1e-5 * abs(ref)


def test_tile_layout_edm_full_size(sm, orc):
    """n = 70000 EDM (2.45e9 pairs) in the E29 layout: streaming checksums of
    the whole output against the oracle's walk of the same layout."""
    n = 70000
    p = workloads.points(n, workloads.SEED_C2)
    plan = sm.smap_plan(2, n, 128, map="below", granularity="tile", layout="tiles")
    out, st = run(sm, plan, "edm", points=dev(p), flags=sm.RUN_CHECKSUM_MIX)
    cs = orc.cs_below_tiles("edm", 2, False, n, 128, points=p)
    assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])
    del out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("m,n,rho", [(2, 1000, 16), (2, 3001, 32), (2, 100, 8), (3, 300, 8), (3, 45, 4), (3, 129, 8)])
@pytest.mark.parametrize("diag", ["strict", "inclusive"])
def test_thread_granularity(sm, orc, m, n, rho, diag):
    """The paper's launch (rho^m threads per block) over the below
    decomposition: same block records, exact cover, index write."""
    plan = sm.smap_plan(m, n, rho, map="below", diag=diag, granularity="thread")
    nint = n + 2 if (m == 3 and diag == "inclusive") else n
    out, _ = run(sm, plan, "map_dump")
    np.testing.assert_array_equal(out.cpu().numpy().reshape(-1, 4), orc.below_tiles(m, -(-nint // rho)))
    out, _ = run(sm, plan, "hitcount", zero=True)
    assert bool((out == 1).all())
    out, st = run(sm, plan, "index_write", flags=sm.RUN_CHECKSUM_MIX)
    exp = orc.index_write(m, diag == "inclusive", n)
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), exp)
    cs = orc.cs_array(exp)
    assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])


@pytest.mark.parametrize("n,rho", [(300, 8), (250, 4), (129, 8)])
def test_thread_granularity_payloads(sm, orc, n, rho):
    p = workloads.points(n, workloads.SEED_C3)
    dp = dev(p)
    plan = sm.smap_plan(3, n, rho, map="below", granularity="thread")
    V = math.comb(n, 3)
    ref = orc.atm_sum(p, np.float32(1e-2))
    _, st = run(sm, plan, "atm", points=dp, param=1e-2)
    assert st["count"] == V and abs(st["sum"] - ref) <= 1e-5 * abs(ref)
    _, st = run(sm, plan, "tc", points=dp, param=0.5)
    assert st["count"] == V and st["tc"] == orc.tc_count(p, np.float32(0.5))
    p2 = workloads.points(1000, workloads.SEED_C2)
    plan2 = sm.smap_plan(2, 1000, 16, map="below", granularity="thread")
    out, _ = run(sm, plan2, "edm", points=dev(p2), flags=sm.RUN_XOR)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), orc.edm(p2).view(np.uint32))
