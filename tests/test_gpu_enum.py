"""GPU parity of the enumeration-map baseline (SMAP_MAP_ENUM, SURVEY NEXT-2;
P:166-174): the block is found from the linear block id by an fp32
square root (m=2) or cube root + square root (m=3) with exact integer
correction.  Compared with the oracle (which walks the rows, no roots) block
by block, thread by thread and element by element; plus an exact cover at
the largest grid one launch allows, where the fp32 roots are least accurate."""
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


@pytest.mark.parametrize("diag", ["strict", "inclusive"])
def test_enum_map_dump_m2(sm, orc, diag):
    for n, rho in [(8, 4), (64, 4), (4096, 4), (16384, 16)]:
        plan = sm.smap_plan(2, n, rho, map="enum", diag=diag)
        out, _ = run(sm, plan, "map_dump")
        np.testing.assert_array_equal(out.cpu().numpy().reshape(-1, 4),
                                      orc.map_dump(2, diag == "inclusive", "enum", n // rho))


def test_enum_map_dump_m3(sm, orc):
    for n, rho in [(16, 2), (64, 2), (512, 2), (1024, 8)]:
        plan = sm.smap_plan(3, n, rho, map="enum")
        out, _ = run(sm, plan, "map_dump")
        np.testing.assert_array_equal(out.cpu().numpy().reshape(-1, 4), orc.map_dump(3, False, "enum", n // rho))


def test_enum_map_dump_large_closed_form(sm):
    # n = 2^13, rho = 1: 33.5M blocks (m=2), bids up to 2^25 where the fp32 root needs the correction
    n = 1 << 13
    plan = sm.smap_plan(2, n, 1, map="enum")
    out, _ = run(sm, plan, "map_dump")
    d = out.view(-1, 4)
    I = torch.repeat_interleave(torch.arange(n, device="cuda"), torch.arange(1, n + 1, device="cuda"))
    bid = torch.arange(len(I), device="cuda")
    J = bid - I * (I + 1) // 2
    assert torch.equal(d[:, 1].long(), I) and torch.equal(d[:, 0].long(), J)
    # m=3, n = 512, rho = 1: 22.5M blocks
    n = 512
    plan = sm.smap_plan(3, n, 1, map="enum")
    out, _ = run(sm, plan, "map_dump")
    d = out.view(-1, 4).cpu().numpy().astype(np.int64)
    I, J, K = d[:, 0], d[:, 1], d[:, 2]
    assert (I <= J).all() and (J <= K).all() and (K < n).all()
    rank = K * (K + 1) * (K + 2) // 6 + J * (J + 1) // 2 + I
    np.testing.assert_array_equal(rank, np.arange(len(d)))


@pytest.mark.parametrize("m,n,rho", [(2, 256, 16), (2, 64, 4), (3, 64, 4), (3, 128, 8)])
def test_enum_thread_dump(sm, orc, m, n, rho):
    for diag in (("strict", "inclusive") if m == 2 else ("strict",)):
        plan = sm.smap_plan(m, n, rho, map="enum", diag=diag)
        out, _ = run(sm, plan, "thread_dump")
        np.testing.assert_array_equal(out.cpu().numpy().view(np.uint64),
                                      orc.thread_dump(m, diag == "inclusive", "enum", n, rho))


@pytest.mark.parametrize("m,n,rho,diag", [(2, 1024, 16, "strict"), (2, 1024, 16, "inclusive"), (3, 256, 8, "strict"),
                                          (2, 1 << 16, 2, "strict"), (3, 1024, 1, "strict")])
def test_enum_hitcount_exact_cover(sm, m, n, rho, diag):
    # (2, 2^16, 2): 536,887,296 blocks, bids up to 2^29; (3, 1024, 1): 179M blocks through the cube root
    plan = sm.smap_plan(m, n, rho, map="enum", diag=diag)
    out, _ = run(sm, plan, "hitcount", zero=True)
    assert out.numel() == sm.smap_volume(m, n, diag)
    assert bool((out == 1).all()), f"missing {(out == 0).sum().item()} duplicated {(out > 1).sum().item()}"


@pytest.mark.parametrize("rho", [8, 16, 32])
@pytest.mark.parametrize("diag", ["strict", "inclusive"])
def test_enum_index_write_m2(sm, orc, rho, diag):
    n = 2048
    plan = sm.smap_plan(2, n, rho, map="enum", diag=diag)
    out, st = run(sm, plan, "index_write", flags=sm.RUN_CHECKSUM_MIX)
    exp = orc.index_write(2, diag == "inclusive", n)
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), exp)
    cs = orc.cs_array(exp)
    assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])


@pytest.mark.parametrize("rho", [4, 8])
def test_enum_index_write_m3(sm, orc, rho):
    n = 256
    plan = sm.smap_plan(3, n, rho, map="enum")
    flags = sm.RUN_CHECKSUM_MIX if rho ** 3 % 32 == 0 else 0
    out, st = run(sm, plan, "index_write", flags=flags)
    exp = orc.index_write(3, False, n)
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), exp)
    if flags:
        cs = orc.cs_array(exp)
        assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])


@pytest.mark.parametrize("rho", [16, 32])
def test_enum_edm_bit_exact(sm, orc, rho):
    n = 2048
    p = workloads.points(n, workloads.SEED_C2)
    plan = sm.smap_plan(2, n, rho, map="enum")
    exp = orc.edm(p)
    cs = orc.cs_array(exp)
    for flags in (0, sm.RUN_XOR, sm.RUN_CHECKSUM_MIX):
        out, st = run(sm, plan, "edm", points=torch.from_numpy(p).cuda(), flags=flags)
        assert np.array_equal(out.cpu().numpy().view(np.uint32), exp.view(np.uint32)), flags
        if flags == sm.RUN_XOR:
            assert (st["count"], st["xr"]) == (cs["count"], cs["xr"])
        if flags == sm.RUN_CHECKSUM_MIX:
            assert (st["count"], st["s0"], st["s1"], st["mix"]) == (cs["count"], cs["s0"], cs["s1"], cs["mix"])


@pytest.mark.parametrize("eps2", [1e-2, 0.0])
def test_enum_atm_sum(sm, orc, eps2):
    n = 256
    p = workloads.points(n, workloads.SEED_C3)
    plan = sm.smap_plan(3, n, 8, map="enum")
    _, st = run(sm, plan, "atm", points=torch.from_numpy(p).cuda(), param=eps2)
    ref = orc.atm_sum(p, np.float32(eps2))
    assert st["count"] == math.comb(n, 3)
    assert abs(st["sum"] - ref) <= 1e-5 * abs(ref)


@pytest.mark.parametrize("R", [0.5, 0.0, 10.0])
def test_enum_tc_count(sm, orc, R):
    n = 256
    p = workloads.points(n, workloads.SEED_C5)
    plan = sm.smap_plan(3, n, 8, map="enum")
    _, st = run(sm, plan, "tc", points=torch.from_numpy(p).cuda(), param=R)
    assert st["count"] == math.comb(n, 3)
    assert st["tc"] == orc.tc_count(p, np.float32(R))


def test_enum_plan_rules(sm):
    plan = sm.smap_plan(2, 1024, 16, map="enum")
    q = sm.smap_plan_query(plan) if hasattr(sm, "smap_plan_query") else None
    if q is not None:
        assert q["grid_blocks"] == 64 * 65 // 2
        assert q["launched_threads"] == 64 * 65 // 2 * 256
    with pytest.raises(Exception):
        sm.smap_plan(2, 1024, 64, map="enum", granularity="tile")
    with pytest.raises(Exception):
        sm.smap_plan(2, 1024, 16, map="enum", shard_rank=0, shard_count=2)
