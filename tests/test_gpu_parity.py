"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle,
element by element on seeded inputs, at sizes that span several tiles and the
diagonal/ragged cases, for both maps and both granularities.  Bar: bit-exact
for coordinates, ranks, indices, counts and fp32 EDM; 1e-5 relative for the
ATM sum (north_star)."""
import math

import numpy as np
import pytest

import workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

MAX64 = np.iinfo(np.uint64).max


@pytest.fixture(scope="module")
def sm():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1610_07394_b200 as s
    return s


def dev_points(p):
    return torch.from_numpy(np.ascontiguousarray(p)).cuda()


def run(sm, plan, payload, points=None, param=0.0, flags=0, zero=False):
    out = sm.alloc_out(plan, payload, zero=zero)
    sm.smap_run(plan, payload, points=points, param=param, out=out, flags=flags)
    st = sm.smap_stats_fetch(plan)
    return out, st


def u64(t):
    return t.cpu().numpy().view(np.uint64)


def u32(t):
    return t.cpu().numpy().view(np.uint32)


# ---------------------------------------------------------------- block maps (a2, a3)
@pytest.mark.parametrize("gran,rho,ns", [("thread", 4, [8, 16, 64, 512, 4096]), ("tile", 32, [64, 256, 2048])])
@pytest.mark.parametrize("map_", ["lambda", "bb"])
@pytest.mark.parametrize("diag", ["strict", "inclusive"])
@pytest.mark.parametrize("order", ["rows", "squares"])
def test_map_dump_m2(sm, orc, gran, rho, ns, map_, diag, order):
    for n in ns:
        plan = sm.smap_plan(2, n, rho, map=map_, diag=diag, granularity=gran, order=order)
        out, _ = run(sm, plan, "map_dump")
        exp = orc.map_dump(2, diag == "inclusive", map_ == "bb", n // rho, order=order)
        np.testing.assert_array_equal(out.cpu().numpy().reshape(-1, 4), exp)


@pytest.mark.parametrize("gran,rho,ns", [("thread", 2, [16, 32, 64, 128, 256, 512]), ("tile", 8, [64, 256, 1024])])
@pytest.mark.parametrize("map_", ["lambda", "bb"])
def test_map_dump_m3(sm, orc, gran, rho, ns, map_):
    for n in ns:
        if map_ == "bb" and (n // rho) > 128:
            continue
        plan = sm.smap_plan(3, n, rho, map=map_, granularity=gran)
        out, _ = run(sm, plan, "map_dump")
        exp = orc.map_dump(3, False, map_ == "bb", n // rho)
        np.testing.assert_array_equal(out.cpu().numpy().reshape(-1, 4), exp)


@pytest.mark.parametrize("G", [2, 4, 8])
def test_map_dump_sharded(sm, orc, G):
    for m, n, rho, order in [(2, 256, 4, "rows"), (2, 256, 4, "squares"), (2, 64, 1, "squares"), (3, 128, 2, "rows")]:
        for r in range(G):
            plan = sm.smap_plan(m, n, rho, shard_rank=r, shard_count=G, order=order)
            out, _ = run(sm, plan, "map_dump")
            exp = orc.map_dump(m, False, False, n // rho, rank=r, G=G, order=order)
            np.testing.assert_array_equal(out.cpu().numpy().reshape(-1, 4), exp)


# ---------------------------------------------------------------- thread -> element (a4, a5)
CASES2 = [(16, 4), (64, 8), (256, 16), (512, 32), (1024, 16)]
CASES3 = [(16, 2), (64, 4), (64, 8), (128, 8), (256, 8)]


@pytest.mark.parametrize("n,rho", CASES2)
@pytest.mark.parametrize("map_", ["lambda", "bb"])
@pytest.mark.parametrize("diag", ["strict", "inclusive"])
@pytest.mark.parametrize("order", ["rows", "squares"])
def test_thread_dump_m2(sm, orc, n, rho, map_, diag, order):
    plan = sm.smap_plan(2, n, rho, map=map_, diag=diag, order=order)
    out, _ = run(sm, plan, "thread_dump")
    np.testing.assert_array_equal(u64(out), orc.thread_dump(2, diag == "inclusive", map_ == "bb", n, rho,
                                                              order=order))


@pytest.mark.parametrize("n,rho", CASES3)
@pytest.mark.parametrize("map_", ["lambda", "bb"])
def test_thread_dump_m3(sm, orc, n, rho, map_):
    plan = sm.smap_plan(3, n, rho, map=map_)
    out, _ = run(sm, plan, "thread_dump")
    np.testing.assert_array_equal(u64(out), orc.thread_dump(3, False, map_ == "bb", n, rho))


def _hit_cases():
    for gran, m, n, rho in [("thread", 2, 1024, 16), ("thread", 2, 64, 4), ("tile", 2, 4096, 128), ("tile", 2, 2048, 64),
                            ("tile", 2, 64, 32), ("thread", 3, 256, 8), ("thread", 3, 64, 2), ("tile", 3, 256, 32),
                            ("tile", 3, 256, 16), ("tile", 3, 128, 8)]:
        for map_ in ("lambda", "bb"):
            for diag in (("strict", "inclusive") if m == 2 else ("strict",)):
                yield gran, m, n, rho, map_, diag


@pytest.mark.parametrize("gran,m,n,rho,map_,diag", list(_hit_cases()))
def test_hitcount_exact_cover(sm, gran, m, n, rho, map_, diag):
    plan = sm.smap_plan(m, n, rho, map=map_, diag=diag, granularity=gran)
    out, _ = run(sm, plan, "hitcount", zero=True)
    h = out.cpu().numpy()
    assert len(h) == sm.smap_volume(m, n, diag)
    assert (h == 1).all(), f"missing {(h == 0).sum()} duplicated {(h > 1).sum()}"


# ---------------------------------------------------------------- payloads (a6) + reductions (a7)
@pytest.mark.parametrize("gran,rho", [("thread", 16), ("thread", 8), ("tile", 32), ("tile", 64), ("tile", 128)])
@pytest.mark.parametrize("map_", ["lambda", "bb"])
@pytest.mark.parametrize("diag", ["strict", "inclusive"])
def test_index_write_m2(sm, orc, gran, rho, map_, diag):
    n = 2048
    plan = sm.smap_plan(2, n, rho, map=map_, diag=diag, granularity=gran)
    out, st = run(sm, plan, "index_write", flags=sm.RUN_CHECKSUM_MIX)
    exp = orc.index_write(2, diag == "inclusive", n)
    np.testing.assert_array_equal(u32(out), exp)
    cs = orc.cs_array(exp)
    assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])
    _, st = run(sm, plan, "index_write", flags=sm.RUN_XOR)
    assert (st["count"], st["xr"]) == (cs["count"], cs["xr"])


@pytest.mark.parametrize("gran,rho", [("thread", 8), ("thread", 4), ("tile", 8), ("tile", 16), ("tile", 32)])
@pytest.mark.parametrize("map_", ["lambda", "bb"])
def test_index_write_m3(sm, orc, gran, rho, map_):
    n = 256
    plan = sm.smap_plan(3, n, rho, map=map_, granularity=gran)
    flags = sm.RUN_CHECKSUM_MIX if (gran == "tile" or rho ** 3 % 32 == 0) else 0
    out, st = run(sm, plan, "index_write", flags=flags)
    exp = orc.index_write(3, False, n)
    np.testing.assert_array_equal(u32(out), exp)
    if flags:
        cs = orc.cs_array(exp)
        assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])


@pytest.mark.parametrize("gran,rho", [("thread", 16), ("thread", 32), ("tile", 32), ("tile", 64), ("tile", 128),
                                      ("tile", 256)])
@pytest.mark.parametrize("map_", ["lambda", "bb"])
@pytest.mark.parametrize("pts", ["uniform", "duplicates", "tiny", "huge"])
def test_edm_bit_exact(sm, orc, gran, rho, map_, pts):
    """Bit-exact fp32 EDM, with and without the fused checksum (different kernel
    paths).  Edge inputs: exact duplicates (r^2 = 0), tiny coordinates (r^2
    below the fast-sqrt range, denormal squares) and huge coordinates (r^2
    overflow to inf) exercise the exact-path fallbacks."""
    n = 2048
    if pts == "uniform":
        p = workloads.points(n, workloads.SEED_C2)
    elif pts == "duplicates":
        p = workloads.clustered_points(n, 5)
    elif pts == "tiny":
        p = (workloads.points(n, 6) * np.float32(1e-30)).astype(np.float32)
    else:
        p = workloads.points(n, 8)
        p[::97] *= np.float32(3e19)
    plan = sm.smap_plan(2, n, rho, map=map_, granularity=gran)
    exp = orc.edm(p)
    cs = orc.cs_array(exp)
    for flags in (0, sm.RUN_XOR, sm.RUN_CHECKSUM, sm.RUN_CHECKSUM_MIX):
        out, st = run(sm, plan, "edm", points=dev_points(p), flags=flags)
        got = out.cpu().numpy()
        assert np.array_equal(got.view(np.uint32), exp.view(np.uint32)), \
            f"flags={flags}: {(got.view(np.uint32) != exp.view(np.uint32)).sum()} mismatching elements"
        if flags:
            assert st["count"] == cs["count"], flags
        if flags == sm.RUN_XOR:
            assert st["xr"] == cs["xr"]
        if flags & (sm.RUN_CHECKSUM | sm.RUN_CHECKSUM_MIX):
            assert (st["s0"], st["s1"]) == (cs["s0"], cs["s1"]), flags
        if flags & sm.RUN_CHECKSUM_MIX:
            assert st["mix"] == cs["mix"]


@pytest.mark.parametrize("gran,rho", [("thread", 8), ("tile", 8), ("tile", 16), ("tile", 32)])
@pytest.mark.parametrize("map_", ["lambda", "bb"])
@pytest.mark.parametrize("eps2", [1e-2, 0.0])
def test_atm_sum(sm, orc, gran, rho, map_, eps2):
    n = 256
    p = workloads.points(n, workloads.SEED_C3)
    plan = sm.smap_plan(3, n, rho, map=map_, granularity=gran)
    _, st = run(sm, plan, "atm", points=dev_points(p), param=eps2)
    ref = orc.atm_sum(p, np.float32(eps2))
    assert st["count"] == math.comb(n, 3)
    assert abs(st["sum"] - ref) <= 1e-5 * abs(ref), (st["sum"], ref)


@pytest.mark.parametrize("gran,rho", [("thread", 8), ("tile", 8), ("tile", 16), ("tile", 32)])
@pytest.mark.parametrize("map_", ["lambda", "bb"])
@pytest.mark.parametrize("R", [0.5, 0.2, 10.0, 0.0])
def test_tc_count(sm, orc, gran, rho, map_, R):
    n = 256
    p = workloads.points(n, workloads.SEED_C5)
    plan = sm.smap_plan(3, n, rho, map=map_, granularity=gran)
    _, st = run(sm, plan, "tc", points=dev_points(p), param=R)
    assert st["count"] == math.comb(n, 3)
    assert st["tc"] == orc.tc_count(p, np.float32(R))


def test_atm_deterministic(sm):
    n = 512
    p = dev_points(workloads.points(n, 3))
    for gran, rho in [("thread", 8), ("tile", 32)]:
        plan = sm.smap_plan(3, n, rho, granularity=gran)
        sums = set()
        for _ in range(3):
            _, st = run(sm, plan, "atm", points=p, param=1e-2)
            sums.add(st["sum"])
        assert len(sums) == 1


# ---------------------------------------------------------------- sharding (a8 host logic, emulated on 1 GPU)
@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("gran,m,n,rho", [("thread", 2, 1024, 16), ("tile", 2, 4096, 64), ("thread", 3, 256, 8),
                                          ("tile", 3, 512, 16)])
def test_shards_partition_exactly(sm, G, gran, m, n, rho):
    hits = None
    tot = {"count": 0, "s0": 0, "s1": 0, "mix": 0}
    for r in range(G):
        plan = sm.smap_plan(m, n, rho, granularity=gran, shard_rank=r, shard_count=G)
        out = sm.alloc_out(plan, "hitcount", zero=True) if hits is None else hits
        sm.smap_run(plan, "hitcount", out=out)
        hits = out
        o2, st = run(sm, plan, "index_write", flags=sm.RUN_CHECKSUM_MIX)
        assert st["count"] == sm.smap_volume(m, n) // G          # exact volume balance (8e)
        for k in tot:
            tot[k] = (tot[k] + st[k]) % (1 << 64)
    assert (hits.cpu().numpy() == 1).all()
    plan = sm.smap_plan(m, n, rho, granularity=gran)
    _, st = run(sm, plan, "index_write", flags=sm.RUN_CHECKSUM_MIX)
    assert all(st[k] == tot[k] for k in tot)


# ---------------------------------------------------------------- device result record + host-buffer API
def test_result_reduce_and_run_host(sm, orc):
    n = 1024
    p = workloads.points(n, 4)
    exp = orc.cs_array(orc.edm(p))
    plan = sm.smap_plan(2, n, 128, granularity="tile")
    out = sm.alloc_out(plan, "edm")
    sm.smap_run(plan, "edm", points=dev_points(p), out=out, flags=sm.RUN_CHECKSUM_MIX)
    rec = torch.zeros(7, dtype=torch.int64, device="cuda")
    sm.smap_result_reduce(plan, rec)
    r = sm.result_dict(rec)
    assert (r["count"], r["s0"], r["s1"], r["mix"]) == (exp["count"], exp["s0"], exp["s1"], exp["mix"])
    pinned = torch.from_numpy(p).pin_memory()
    out.zero_()
    st = sm.smap_run_host(plan, "edm", host_points=pinned, out=out, flags=sm.RUN_CHECKSUM)
    assert (st["count"], st["s0"], st["s1"]) == (exp["count"], exp["s0"], exp["s1"])
    assert st["launches"] == 2
    # ATM through the record: fp64 field
    p3 = workloads.points(128, 5)
    plan3 = sm.smap_plan(3, 128, 16, granularity="tile")
    st3 = sm.smap_run_host(plan3, "atm", host_points=p3, param=1e-2)
    ref = orc.atm_sum(p3, np.float32(1e-2))
    assert abs(st3["sum"] - ref) <= 1e-5 * abs(ref)


# ---------------------------------------------------------------- closed forms vs launch
@pytest.mark.parametrize("m,n,rho,map_,diag,launched,useful", [
    (2, 1024, 16, "lambda", "strict", 1024 * 1024 // 2, 1024 * 1023 // 2),
    (2, 1024, 16, "lambda", "inclusive", 1024 * (1024 + 16) // 2, 1024 * 1025 // 2),
    (2, 1024, 16, "bb", "strict", 1024 ** 2, 1024 * 1023 // 2),
    (3, 1024, 8, "lambda", "strict", 3 * 1024 ** 3 // 16, math.comb(1024, 3)),
    (3, 1024, 8, "bb", "strict", 1024 ** 3, math.comb(1024, 3)),
])
def test_plan_closed_forms(sm, m, n, rho, map_, diag, launched, useful):
    q = sm.smap_plan_query(sm.smap_plan(m, n, rho, map=map_, diag=diag))
    assert q["launched_threads"] == launched and q["useful_elems"] == useful
    assert q["wasted_threads"] == launched - useful


# ---------------------------------------------------------------- edge cases / errors
def test_smallest_grids(sm, orc):
    for m, n, rho in [(2, 2, 1), (2, 8, 4), (3, 8, 1), (3, 16, 2)]:
        plan = sm.smap_plan(m, n, rho)
        out, _ = run(sm, plan, "hitcount", zero=True)
        assert (out.cpu().numpy() == 1).all()


def test_invalid_arguments(sm):
    bad = [dict(m=4, n=64, rho=8), dict(m=2, n=100, rho=3), dict(m=2, n=64, rho=128), dict(m=2, n=1, rho=1),
           dict(m=3, n=32, rho=8), dict(m=3, n=2, rho=1), dict(m=2, n=64, rho=8, shard_count=3),
           dict(m=2, n=64, rho=8, shard_count=8), dict(m=2, n=64, rho=8, map="bb", shard_count=2),
           dict(m=2, n=1024, rho=16, granularity="tile"), dict(m=2, n=1024, rho=16, persistent=2)]
    for kw in bad:
        with pytest.raises(sm.SmapError) as e:
            sm.smap_plan(**kw)
        assert e.value.status == 1, kw
    plan = sm.smap_plan(2, 256, 16)
    small = torch.empty(10, dtype=torch.int32, device="cuda")
    with pytest.raises(sm.SmapError):
        sm.smap_run(plan, "index_write", out=small)
    with pytest.raises(sm.SmapError):
        sm.smap_run(plan, "atm", out=None)        # m=3 payload on an m=2 plan
    with pytest.raises(sm.SmapError):
        sm.smap_run(plan, "edm", out=sm.alloc_out(plan, "edm"))   # no points


def test_run_rejects_bad_buffers(sm):
    """Boundary checks of smap_run (include/smap.h): short or misaligned
    buffers are SMAP_E_INVALID before any launch; the binding refuses host
    arrays, wrong dtypes and raw pointers without a size."""
    import ctypes as C
    n = 1024
    plan = sm.smap_plan(2, n, 128, granularity="tile", layout="tiles")
    pts = torch.from_numpy(workloads.points(n, 1)).cuda()
    out = sm.alloc_out(plan, "edm")
    with pytest.raises(sm.SmapError) as e:                      # one point short (the r01 initcheck case)
        sm.smap_run(plan, "edm", points=pts.data_ptr(), points_bytes=(n - 1) * 12, out=out)
    assert e.value.status == sm.E_INVALID and "points" in str(e.value)
    big = torch.empty(out.numel() + 4, dtype=torch.float32, device="cuda")
    with pytest.raises(sm.SmapError) as e:                      # 4-B aligned out on a 16-B vector-store layout
        sm.smap_run(plan, "edm", points=pts, out=big.data_ptr() + 4, out_bytes=out.numel() * 4)
    assert e.value.status == sm.E_INVALID and "aligned" in str(e.value)
    with pytest.raises(TypeError):                              # host arrays belong to smap_run_host
        sm.smap_run(plan, "edm", points=workloads.points(n, 1), out=out)
    with pytest.raises(ValueError):
        sm.smap_run(plan, "edm", points=pts.double(), out=out)
    with pytest.raises(ValueError):
        sm.smap_run(plan, "edm", points=pts[: n // 2], out=out)
    with pytest.raises(ValueError):
        sm.smap_run(plan, "edm", points=pts, out=out.data_ptr())   # raw pointer without out_bytes
    with pytest.raises(ValueError):
        sm.smap_run_host(plan, "edm", host_points=pts, out=out)   # device tensor given as host points
    with pytest.raises(sm.SmapError):
        sm._lib.smap_run_host(plan.handle, sm.PAYLOAD["edm"], C.c_void_p(workloads.points(n, 1).ctypes.data),
                              12 * n - 12, 0.0, C.c_void_p(out.data_ptr()), out.numel() * 4, 0, None,
                              C.byref(sm.Stats())) and sm._check(sm.E_INVALID)
    # the plan still runs after the rejected calls
    sm.smap_run(plan, "edm", points=pts, out=out, flags=sm.RUN_XOR)
    assert sm.smap_stats_fetch(plan)["count"] == n * (n - 1) // 2


# ---------------------------------------------------------------- m=3 tiles of 64 (TC / index write / cover)
@pytest.mark.parametrize("map_", ["lambda", "bb"])
def test_tile64_m3(sm, orc, map_):
    """rho = 64 m=3 tiles (64-bit predicate rows for TC; two lane chunks per
    row in the index walker): exact cover, index write in both layouts, TC
    count against the oracle, the map dump; ATM is rejected (smem tables)."""
    n = 512 if map_ == "lambda" else 256
    plan = sm.smap_plan(3, n, 64, map=map_, granularity="tile")
    out, _ = run(sm, plan, "hitcount", zero=True)
    assert (out.cpu().numpy() == 1).all()
    out, _ = run(sm, plan, "map_dump")
    np.testing.assert_array_equal(out.cpu().numpy().reshape(-1, 4), orc.map_dump(3, False, map_ == "bb", n // 64))
    iw = orc.index_write(3, False, n)
    out, st = run(sm, plan, "index_write", flags=sm.RUN_CHECKSUM_MIX)
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), iw)
    plan_t = sm.smap_plan(3, n, 64, map=map_, granularity="tile", layout="tiles")
    out, st = run(sm, plan_t, "index_write", flags=sm.RUN_XOR)
    exp = orc.to_tile_layout3(iw, n, 64, map_ == "bb")
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), exp)
    cs = orc.cs_array(exp)
    assert (st["count"], st["xr"]) == (cs["count"], cs["xr"])
    p = workloads.points(n, workloads.SEED_C5)
    for R in (0.5, 0.2, 10.0):
        _, st = run(sm, plan, "tc", points=dev_points(p), param=R)
        assert st["count"] == math.comb(n, 3)
        assert st["tc"] == orc.tc_count(p, np.float32(R))
    with pytest.raises(sm.SmapError):
        sm.smap_run(plan, "atm", points=dev_points(p), param=1e-2)


@pytest.mark.parametrize("G", [1, 2, 8, 33])
def test_result_combine_kernel(sm, G):
    """smap_result_combine (the bench's cross-rank step after the all-gather)
    equals the plain combination: integer fields mod 2^64, xor, fp64 sums in
    record order."""
    import bench
    rng = np.random.default_rng(G)
    recs = rng.integers(-(1 << 63), (1 << 63) - 1, size=(G, 7), dtype=np.int64)
    recs[:, 6] = rng.standard_normal(G).view(np.int64)
    d = torch.from_numpy(recs).cuda()
    out = torch.zeros(7, dtype=torch.int64, device="cuda")
    sm.smap_result_combine(d, G, out)
    exp = bench.combine_records(torch.from_numpy(recs))
    got = out.cpu()
    assert torch.equal(got[:6], exp[:6])
    s = 0.0
    for g in range(G):
        s += float(recs[g, 6:7].view(np.float64)[0])
    assert float(got[6:7].numpy().view(np.float64)[0]) == s
    sm.smap_result_combine(d, G, d[0])                  # dst may alias records[0]
    assert torch.equal(d[0].cpu()[:6], exp[:6])


def test_c_example_runs(tmp_path):
    """examples/edm_c_api.c run as a C program on the GPU: exit 0 means the
    count and one located distance matched its own fp32 recomputation."""
    import subprocess
    import test_abi
    exe = test_abi._build_c_example(tmp_path)
    r = subprocess.run([exe, "3000"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("gran,rho", [("thread", 8), ("tile", 16), ("tile", 32)])
@pytest.mark.parametrize("map_", ["lambda", "below"])
def test_atm_tc_degenerate_points(sm, orc, gran, rho, map_):
    """Degenerate point sets: exact duplicates (r^2 = 0, softened by eps^2 for
    ATM; always inside R for TC) and a tiny-scale cloud (r^2 near the fp32
    denormal range) -- the packed ATM path falls back to the IEEE-ordered term
    where its partial is not finite; TC compares the same fp32 r^2."""
    n = 256
    for p in (workloads.clustered_points(n, 21), (workloads.points(n, 22) * np.float32(1e-12)).astype(np.float32)):
        dp = dev_points(p)
        plan = sm.smap_plan(3, n, rho, map=map_, granularity=gran)
        _, st = run(sm, plan, "atm", points=dp, param=1e-2)
        ref = orc.atm_sum(p, np.float32(1e-2))
        assert st["count"] == math.comb(n, 3)
        assert abs(st["sum"] - ref) <= 1e-5 * abs(ref), (st["sum"], ref)
        for R in (0.5, 1e-12, 0.0):
            _, st = run(sm, plan, "tc", points=dp, param=R)
            assert st["tc"] == orc.tc_count(p, np.float32(R)), R
