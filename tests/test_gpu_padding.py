"""GPU parity for any n ("approach n from above")
and the inclusive tetrahedron (reading E24): non-power-of-two n through every
kernel family -- thread dumps, exact covers, index write with checksums,
bit-exact EDM (cut tiles take the exact row walker), ATM and TC -- against
the oracle on the same seeded inputs."""
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


@pytest.mark.parametrize("m,n,rho,diag", [(2, 1000, 16, "strict"), (2, 777, 8, "inclusive"), (2, 3, 2, "strict"),
                                          (3, 100, 4, "strict"), (3, 61, 4, "inclusive"), (3, 200, 8, "strict")])
@pytest.mark.parametrize("map_", ["lambda", "bb", "enum"])
def test_padded_thread_dump(sm, orc, m, n, rho, diag, map_):
    nint = n + 2 if (m == 3 and diag == "inclusive") else n
    N = orc.padded_n(nint) // rho
    if map_ == "lambda" and ((m == 2 and N < 2) or (m == 3 and N < 8)):
        pytest.skip("grid below lambda's minimum")
    plan = sm.smap_plan(m, n, rho, map=map_, diag=diag)
    out, _ = run(sm, plan, "thread_dump")
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint64),
                                  orc.thread_dump(m, diag == "inclusive", map_, n, rho))


def _cover_cases():
    for gran, m, n, rho in [("thread", 2, 1000, 16), ("thread", 2, 100001, 32), ("tile", 2, 1000, 32),
                            ("tile", 2, 5000, 128), ("tile", 2, 70000, 256), ("thread", 3, 300, 8), ("thread", 3, 37, 2),
                            ("tile", 3, 300, 8), ("tile", 3, 1000, 32), ("tile", 3, 500, 16)]:
        for map_ in ("lambda", "bb"):
            for diag in ("strict", "inclusive"):
                yield gran, m, n, rho, map_, diag
    for m, n, rho in [(2, 3000, 16), (3, 250, 8)]:
        for diag in ("strict", "inclusive"):
            yield "thread", m, n, rho, "enum", diag


@pytest.mark.parametrize("gran,m,n,rho,map_,diag", list(_cover_cases()))
def test_padded_hitcount_exact_cover(sm, gran, m, n, rho, map_, diag):
    plan = sm.smap_plan(m, n, rho, map=map_, diag=diag, granularity=gran)
    out, _ = run(sm, plan, "hitcount", zero=True)
    assert out.numel() == sm.smap_volume(m, n, diag)
    assert bool((out == 1).all()), f"missing {(out == 0).sum().item()} duplicated {(out > 1).sum().item()}"


@pytest.mark.parametrize("gran,rho", [("thread", 16), ("tile", 32), ("tile", 128), ("tile", 512)])
@pytest.mark.parametrize("map_", ["lambda", "bb"])
@pytest.mark.parametrize("diag", ["strict", "inclusive"])
def test_padded_index_write_m2(sm, orc, gran, rho, map_, diag):
    n = 1500
    plan = sm.smap_plan(2, n, rho, map=map_, diag=diag, granularity=gran)
    out, st = run(sm, plan, "index_write", flags=sm.RUN_CHECKSUM_MIX)
    exp = orc.index_write(2, diag == "inclusive", n)
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), exp)
    cs = orc.cs_array(exp)
    assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])


@pytest.mark.parametrize("gran,rho", [("thread", 8), ("tile", 8), ("tile", 16), ("tile", 32)])
@pytest.mark.parametrize("map_", ["lambda", "bb"])
@pytest.mark.parametrize("diag", ["strict", "inclusive"])
def test_padded_index_write_m3(sm, orc, gran, rho, map_, diag):
    n = 300
    plan = sm.smap_plan(3, n, rho, map=map_, diag=diag, granularity=gran)
    out, st = run(sm, plan, "index_write", flags=sm.RUN_CHECKSUM_MIX)
    exp = orc.index_write(3, diag == "inclusive", n)
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), exp)
    cs = orc.cs_array(exp)
    assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])


@pytest.mark.parametrize("gran,rho", [("thread", 16), ("tile", 32), ("tile", 64), ("tile", 128), ("tile", 256)])
@pytest.mark.parametrize("map_", ["lambda", "bb"])
@pytest.mark.parametrize("n", [1000, 2049])
def test_padded_edm_bit_exact(sm, orc, gran, rho, map_, n):
    p = workloads.points(n, workloads.SEED_C2)
    plan = sm.smap_plan(2, n, rho, map=map_, granularity=gran)
    exp = orc.edm(p)
    cs = orc.cs_array(exp)
    for flags in (0, sm.RUN_XOR, sm.RUN_CHECKSUM):
        out, st = run(sm, plan, "edm", points=dev(p), flags=flags)
        assert np.array_equal(out.cpu().numpy().view(np.uint32), exp.view(np.uint32)), flags
        if flags == sm.RUN_XOR:
            assert (st["count"], st["xr"]) == (cs["count"], cs["xr"])
        if flags == sm.RUN_CHECKSUM:
            assert (st["count"], st["s0"], st["s1"]) == (cs["count"], cs["s0"], cs["s1"])


@pytest.mark.parametrize("gran,rho", [("thread", 8), ("tile", 8), ("tile", 16), ("tile", 32)])
@pytest.mark.parametrize("map_", ["lambda", "bb"])
@pytest.mark.parametrize("n", [200, 333])
def test_padded_atm_and_tc(sm, orc, gran, rho, map_, n):
    p = workloads.points(n, workloads.SEED_C3)
    plan = sm.smap_plan(3, n, rho, map=map_, granularity=gran)
    _, st = run(sm, plan, "atm", points=dev(p), param=1e-2)
    ref = orc.atm_sum(p, np.float32(1e-2))
    assert st["count"] == math.comb(n, 3)
    assert abs(st["sum"] - ref) <= 1e-5 * abs(ref)
    _, st = run(sm, plan, "tc", points=dev(p), param=0.5)
    assert st["count"] == math.comb(n, 3)
    assert st["tc"] == orc.tc_count(p, np.float32(0.5))


def test_inclusive_m3_rejects_point_payloads(sm):
    plan = sm.smap_plan(3, 100, 8, diag="inclusive")
    p = dev(workloads.points(100, 1))
    with pytest.raises(Exception):
        sm.smap_run(plan, "atm", points=p, param=1e-2)
    with pytest.raises(Exception):
        sm.smap_run(plan, "tc", points=p, param=0.5)


@pytest.mark.parametrize("map_", ["lambda", "bb"])
@pytest.mark.parametrize("n", [777, 1000, 1024])
@pytest.mark.parametrize("persistent", [0, 16])
def test_tc_tile64_any_n(sm, orc, map_, n, persistent):
    """The T = 64 TC tiles (128-thread CTAs, double-buffered bit rows, the symmetric
    32 x 32-block bitmap pass) at padded and power-of-two n, persistent or not."""
    p = workloads.points(n, 23)
    plan = sm.smap_plan(3, n, 64, map=map_, granularity="tile", persistent=persistent)
    _, st = run(sm, plan, "tc", points=dev(p), param=0.5)
    assert st["count"] == math.comb(n, 3)
    assert st["tc"] == orc.tc_count(p, np.float32(0.5))


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("rho,persistent", [(64, 16), (64, 32), (32, 8)])
def test_tc_tile64_shards_add_up(sm, orc, G, rho, persistent):
    """Sharded TC plans build only the bitmap blocks their tiles read (the plan's
    shard analysis); the shard counts must still add up to the oracle's count."""
    n = 1024
    p = workloads.points(n, 29)
    tot = cnt = 0
    for r in range(G):
        plan = sm.smap_plan(3, n, rho, granularity="tile", persistent=persistent, shard_rank=r, shard_count=G)
        _, st = run(sm, plan, "tc", points=dev(p), param=0.5)
        tot += st["tc"]
        cnt += st["count"]
    assert cnt == math.comb(n, 3)
    assert tot == orc.tc_count(p, np.float32(0.5))


@pytest.mark.parametrize("map_", ["lambda", "bb"])
@pytest.mark.parametrize("n", [1000, 2048])
def test_tc_tile64_64thread_ctas(sm, orc, map_, n):
    """persistent >= 32 selects the 64-thread TC CTAs (64 k rows per thread)."""
    p = workloads.points(n, 31)
    plan = sm.smap_plan(3, n, 64, map=map_, granularity="tile", persistent=32)
    _, st = run(sm, plan, "tc", points=dev(p), param=0.5)
    assert st["count"] == math.comb(n, 3)
    assert st["tc"] == orc.tc_count(p, np.float32(0.5))
