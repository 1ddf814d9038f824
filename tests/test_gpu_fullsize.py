"""GPU parity at BASELINE.json's full sizes, in the launch configurations that
bench.py times: sampled outputs the oracle computes one by one (located with
smap_locate), plus the order-independent checksums (reading E21) the oracle
streams over the whole domain on the host cores."""
import math

import numpy as np
import pytest

import workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sm():
    assert torch.cuda.is_available()
    import paper_1610_07394_b200 as s
    return s


def _sample_pairs(n, k, seed):
    rng = np.random.default_rng(seed)
    i = rng.integers(1, n, size=k)
    j = (rng.random(k) * i).astype(np.int64)
    # always include the extremes and the diagonal neighbours
    i = np.concatenate([i, [1, n - 1, n - 1, n // 2]])
    j = np.concatenate([j, [0, 0, n - 2, n // 2 - 1]])
    return i, j


def _positions(sm, plan, i, j):
    return np.array([sm.smap_locate(plan, int(a), int(b))[1] for a, b in zip(i, j)], np.int64)


@pytest.mark.parametrize("cfg", workloads.BENCH_EDM_VARIANTS)
def test_c2_edm_full(sm, orc, cfg):
    n = workloads.CONFIGS["C2"]["n"]
    p = workloads.points(n, workloads.SEED_C2)
    plan = sm.smap_plan(2, n, **cfg)
    out = sm.alloc_out(plan, "edm")
    sm.smap_run(plan, "edm", points=torch.from_numpy(p).cuda(), out=out, flags=sm.RUN_CHECKSUM_MIX)
    st = sm.smap_stats_fetch(plan)
    i, j = _sample_pairs(n, 50000, 1)
    pos = torch.from_numpy(_positions(sm, plan, i, j)).cuda()
    got = out[pos].cpu().numpy()
    exp = orc.edm_dist_many(p, i, j)
    assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))
    if cfg.get("layout") == "tiles":
        cs = orc.cs_tiles2("edm", n, cfg["rho"], bb=cfg["map"] == "bb", points=p)
    else:
        cs = orc.cs_edm(p)
    assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])
    del out
    torch.cuda.empty_cache()


def test_c3_index_and_atm_full(sm, orc):
    c = workloads.CONFIGS["C3"]
    n = c["n"]
    p = workloads.points(n, workloads.SEED_C3)
    ref = orc.atm_sum(p, np.float32(c["eps2"]))
    for cfg in workloads.BENCH_M3_VARIANTS:
        plan = sm.smap_plan(3, n, **cfg)
        out = sm.alloc_out(plan, "index_write")
        sm.smap_run(plan, "index_write", out=out, flags=sm.RUN_CHECKSUM)
        st = sm.smap_stats_fetch(plan)
        V = math.comb(n, 3)
        assert st["count"] == V
        got = out.cpu().numpy().view(np.uint32)
        assert np.array_equal(got, np.arange(V, dtype=np.uint32))
        sm.smap_run(plan, "atm", points=torch.from_numpy(p).cuda(), param=c["eps2"])
        st = sm.smap_stats_fetch(plan)
        assert abs(st["sum"] - ref) <= 1e-5 * abs(ref)


def test_c3_index_write_tile_layout_full(sm, orc):
    """C3 index write in the m=3 tile-blocked layout (reading E26): full-size
    streaming checksums against the oracle's enumerated layout, unsharded and
    as 4 shards, plus sampled positions through smap_locate."""
    n = workloads.CONFIGS["C3"]["n"]
    V = math.comb(n, 3)
    for bb, G in ((False, 1), (False, 4), (True, 1)):
        for r in range(G):
            plan = sm.smap_plan(3, n, 32, map="bb" if bb else "lambda", granularity="tile", shard_rank=r,
                                shard_count=G, layout="tiles")
            out = sm.alloc_out(plan, "index_write")
            sm.smap_run(plan, "index_write", out=out, flags=sm.RUN_CHECKSUM_MIX)
            st = sm.smap_stats_fetch(plan)
            cs = orc.cs_tiles3(n, 32, bb, r, G)
            assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])
            assert st["count"] * G == V if not bb else st["count"] == V
            got = out.cpu().numpy().view(np.uint32)
            rng = np.random.default_rng(r)
            for _ in range(2000):
                i, j, k = sorted(int(v) for v in rng.choice(n, 3, replace=False))
                sh, pos = sm.smap_locate(plan, i, j, k)
                if sh == r:
                    assert got[pos] == math.comb(k, 3) + math.comb(j, 2) + i


def test_c5_tc_full(sm, orc):
    c = workloads.CONFIGS["C5"]
    n = c["n"]
    p = workloads.points(n, workloads.SEED_C5)
    ref = orc.tc_count(p, np.float32(c["R"]))
    for cfg in workloads.BENCH_M3_VARIANTS + [dict(rho=64, granularity="tile", map="lambda"), workloads.BENCH_C5]:
        plan = sm.smap_plan(3, n, **cfg)
        sm.smap_run(plan, "tc", points=torch.from_numpy(p).cuda(), param=c["R"])
        st = sm.smap_stats_fetch(plan)
        assert st["count"] == math.comb(n, 3)
        assert st["tc"] == ref


@pytest.mark.parametrize("layout", ["tiles", "rows"])
def test_c4_index_write_full(sm, orc, layout):
    n = workloads.CONFIGS["C4"]["n"]
    V = n * (n - 1) // 2
    cfg = dict(workloads.BENCH_C4, layout=layout)
    plan = sm.smap_plan(2, n, **cfg)
    out = sm.alloc_out(plan, "index_write")             # 68.7 GB of uint64 on the device
    assert out.numel() == V and out.dtype == torch.int64
    sm.smap_run(plan, "index_write", out=out, flags=sm.RUN_CHECKSUM_MIX)
    st = sm.smap_stats_fetch(plan)
    M = 1 << 64
    assert st["count"] == V
    assert st["s0"] == (V * (V - 1) // 2) % M           # values are the canonical ranks in both layouts
    i, j = _sample_pairs(n, 50000, 2)
    rank = i * (i - 1) // 2 + j
    got = out[torch.from_numpy(_positions(sm, plan, i, j)).cuda()].cpu().numpy()
    assert np.array_equal(got, rank)
    if layout == "rows":
        assert st["s1"] == ((V - 1) * V * (V + 1) // 3) % M
        cs = orc.cs_index(2, False, n)
    else:
        cs = orc.cs_tiles2("index_write", n, cfg["rho"])
    assert (st["s1"], st["mix"]) == (cs["s1"], cs["mix"])
    del out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("G", [2, 8])
def test_c4_sharded_tiles_partition(sm, orc, G):
    """Each shard writes a shard-local V/G array; the records add up to the
    unsharded ones (the bench's all-reduce, emulated on one GPU)."""
    n = workloads.CONFIGS["C4"]["n"] // 4           # 2^15: keeps the emulation quick
    V = n * (n - 1) // 2
    tot = [0, 0, 0, 0]
    for r in range(G):
        plan = sm.smap_plan(2, n, shard_rank=r, shard_count=G, **workloads.BENCH_C4)
        out = sm.alloc_out(plan, "index_write")
        assert out.numel() == V // G
        sm.smap_run(plan, "index_write", out=out, flags=sm.RUN_CHECKSUM_MIX)
        st = sm.smap_stats_fetch(plan)
        cs = orc.cs_tiles2("index_write", n, workloads.BENCH_C4["rho"], rank=r, G=G)
        assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])
        tot = [(a + b) % (1 << 64) for a, b in zip(tot, (st["count"], st["s0"], st["s1"], st["mix"]))]
    assert tot[0] == V and tot[1] == (V * (V - 1) // 2) % (1 << 64)


def test_m3_uint64_index_write_full(sm, orc):
    """m=3 with V > 2^32 (n = 3000: 4.5e9 triples, 36 GB of uint64 ranks) through
    the from-below map's E29 tile layout: the u64 tile kernels at full size,
    streaming checksums against the oracle's walk of the same layout."""
    n = 3000
    plan = sm.smap_plan(3, n, 32, map="below", granularity="tile", layout="tiles")
    out = sm.alloc_out(plan, "index_write")
    assert out.dtype == torch.int64
    sm.smap_run(plan, "index_write", out=out, flags=sm.RUN_CHECKSUM_MIX)
    st = sm.smap_stats_fetch(plan)
    cs = orc.cs_below_tiles("index_write", 3, False, n, 32)
    assert st["count"] == math.comb(n, 3) == cs["count"]
    assert (st["s0"], st["s1"], st["mix"]) == (cs["s0"], cs["s1"], cs["mix"])
    del out
    torch.cuda.empty_cache()


def test_m3_index_write_n2048_tiles_full(sm, orc):
    """C5's size (n = 2048, 1.43e9 triples) as an index write in the lambda3
    tile layout (E26) at the bench tile 32: full streaming checksums."""
    n = 2048
    plan = sm.smap_plan(3, n, 32, granularity="tile", layout="tiles")
    out = sm.alloc_out(plan, "index_write")
    sm.smap_run(plan, "index_write", out=out, flags=sm.RUN_CHECKSUM_MIX)
    st = sm.smap_stats_fetch(plan)
    cs = orc.cs_tiles3(n, 32)
    assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])
    del out
    torch.cuda.empty_cache()


def test_m3_uint64_fused_full(sm, orc):
    """The fused index write + ATM with uint64 ranks (V > 2^32 at n = 3000):
    index checksums and the fp64 ATM sum against the oracle."""
    n = 3000
    p = workloads.points(n, workloads.SEED_C3)
    plan = sm.smap_plan(3, n, 32, map="below", granularity="tile", layout="tiles")
    out = sm.alloc_out(plan, "index_write_atm")
    sm.smap_run(plan, "index_write_atm", points=torch.from_numpy(p).cuda(), param=1e-2, out=out,
                flags=sm.RUN_CHECKSUM_MIX)
    st = sm.smap_stats_fetch(plan)
    del out
    torch.cuda.empty_cache()
    cs = orc.cs_below_tiles("index_write", 3, False, n, 32)
    assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])
    ref = orc.atm_sum(p, np.float32(1e-2))
    assert abs(st["sum"] - ref) <= 1e-5 * abs(ref), (st["sum"], ref)


@pytest.mark.parametrize("m,n,rho,mp", [(3, 3000, 8, "lambda"), (3, 3000, 8, "below"), (2, 1 << 17, 16, "lambda"),
                                        (2, 100000, 16, "below")])
def test_uint64_index_write_thread_full(sm, orc, m, n, rho, mp):
    """uint64 ranks at the paper's launch (one element per thread): canonical
    layout, full streaming checksums (m=3 n=3000: 4.5e9 triples; m=2 n=2^17:
    8.6e9 pairs = C4)."""
    plan = sm.smap_plan(m, n, rho, map=mp, granularity="thread")
    out = sm.alloc_out(plan, "index_write")
    assert out.dtype == torch.int64
    sm.smap_run(plan, "index_write", out=out, flags=sm.RUN_CHECKSUM_MIX)
    st = sm.smap_stats_fetch(plan)
    del out
    torch.cuda.empty_cache()
    cs = orc.cs_index(m, False, n)
    assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])
