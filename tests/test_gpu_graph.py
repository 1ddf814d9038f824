"""smap_graph_capture / smap_graph_launch (include/smap.h): a captured step
replays the same kernels as smap_run + smap_result_reduce, so its device
record must equal the direct run's, bit for bit, on every replay; the bound
output buffer must hold the same values.  Checked against the oracle where
the payload has a cheap oracle value."""
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


CASES = [
    (2, 2048, dict(rho=128, granularity="tile", layout="tiles"), "edm", 0.0, "xor"),
    (2, 4096, dict(rho=128, granularity="tile", layout="tiles"), "index_write", 0.0, "checksum"),
    (3, 512, dict(rho=32, granularity="tile", layout="tiles"), "index_write_atm", 1e-2, "none"),
    (3, 512, dict(rho=32, granularity="tile"), "atm", 1e-2, "none"),
    (3, 1024, dict(rho=64, granularity="tile", persistent=8), "tc", 0.5, "none"),
    (3, 256, dict(rho=8, granularity="thread"), "tc", 0.5, "none"),
    (2, 1024, dict(rho=16, granularity="thread"), "edm", 0.0, "mix"),
]


@pytest.mark.parametrize("m,n,kw,payload,param,mode", CASES)
def test_graph_replay_equals_direct_run(sm, orc, m, n, kw, payload, param, mode):
    flags = {"none": 0, "xor": sm.RUN_XOR, "checksum": sm.RUN_CHECKSUM, "mix": sm.RUN_CHECKSUM_MIX}[mode]
    plan = sm.smap_plan(m, n, **kw)
    p = workloads.points(n, 11)
    pts = torch.from_numpy(p).cuda() if payload in ("edm", "atm", "tc", "index_write_atm") else None
    out = sm.alloc_out(plan, payload)
    rec_direct = torch.zeros(7, dtype=torch.int64, device="cuda")
    sm.smap_run(plan, payload, points=pts, param=param, out=out, flags=flags)
    sm.smap_result_reduce(plan, rec_direct)
    direct = sm.result_dict(rec_direct)
    ref_out = out.clone() if out is not None else None
    rec = torch.zeros(7, dtype=torch.int64, device="cuda")
    g = sm.smap_graph_capture(plan, payload, points=pts, param=param, out=out, flags=flags, record=rec)
    assert g.launches >= 2                                      # the payload kernel(s) + the reduction
    if out is not None:
        out.zero_()
    for _ in range(3):
        sm.smap_graph_launch(g)
        torch.cuda.synchronize()
        assert sm.result_dict(rec) == direct
    if out is not None:
        assert torch.equal(out, ref_out)
    V = sm.smap_volume(m, n)
    assert direct["count"] == V
    if payload == "tc":
        assert direct["tc"] == orc.tc_count(p, np.float32(param))
    if payload in ("atm", "index_write_atm"):
        ref = orc.atm_sum(p, np.float32(param))
        assert abs(direct["sum"] - ref) <= 1e-5 * abs(ref)
    if payload == "edm" and flags == sm.RUN_XOR:
        assert direct["xr"] == orc.cs_edm(p)["xr"]


def test_graph_capture_validates(sm):
    plan = sm.smap_plan(2, 1024, 128, granularity="tile", layout="tiles")
    out = sm.alloc_out(plan, "edm")
    with pytest.raises(sm.SmapError):                          # EDM without points: rejected before capture
        sm.smap_graph_capture(plan, "edm", out=out)
    rec = torch.zeros(8, dtype=torch.int64, device="cuda")
    with pytest.raises(sm.SmapError):                          # misaligned record
        sm.smap_graph_capture(plan, "index_write", out=out.view(torch.int32), record=rec.data_ptr() + 4)
    # a stream-ordered replay on a side stream is ordered with the work on that stream
    g = sm.smap_graph_capture(plan, "index_write", out=out.view(torch.int32), flags=sm.RUN_XOR, record=rec)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        sm.smap_graph_launch(g, stream=s)
    s.synchronize()
    assert sm.result_dict(rec)["count"] == math.comb(1024, 2)


@pytest.mark.parametrize("m,n,kw,payload,param,mode", [c for c in CASES if c[2].get("granularity") == "tile"][:5])
def test_graph_interleaved_with_direct_runs(sm, m, n, kw, payload, param, mode):
    """A captured step clears the result block behind its record (no memset node);
    an smap_run in between leaves its results there, and the next replay must
    still start from a clear block: graph, run, graph, run, graph all agree."""
    flags = {"none": 0, "xor": sm.RUN_XOR, "checksum": sm.RUN_CHECKSUM, "mix": sm.RUN_CHECKSUM_MIX}[mode]
    plan = sm.smap_plan(m, n, **kw)
    p = workloads.points(n, 17)
    pts = torch.from_numpy(p).cuda() if payload in ("edm", "atm", "tc", "index_write_atm") else None
    out = sm.alloc_out(plan, payload)
    rec = torch.zeros(7, dtype=torch.int64, device="cuda")
    g = sm.smap_graph_capture(plan, payload, points=pts, param=param, out=out, flags=flags, record=rec)
    results = []
    for step in range(5):
        if step % 2 == 0:
            sm.smap_graph_launch(g)
            torch.cuda.synchronize()
            results.append(sm.result_dict(rec))
        else:
            sm.smap_run(plan, payload, points=pts, param=param, out=out, flags=flags)
            r2 = torch.zeros(7, dtype=torch.int64, device="cuda")
            sm.smap_result_reduce(plan, r2)
            torch.cuda.synchronize()
            results.append(sm.result_dict(r2))
            assert sm.smap_stats_fetch(plan)["count"] == results[-1]["count"]
    assert all(r == results[0] for r in results), results
    assert results[0]["count"] == sm.smap_volume(m, n)


def test_record_buffers_checked_by_the_binding(sm):
    plan = sm.smap_plan(2, 1024, 128, granularity="tile", layout="tiles")
    out = sm.alloc_out(plan, "index_write")
    small = torch.zeros(3, dtype=torch.int64, device="cuda")          # < 56 bytes
    with pytest.raises(ValueError):
        sm.smap_graph_capture(plan, "index_write", out=out, record=small)
    sm.smap_run(plan, "index_write", out=out)
    with pytest.raises(ValueError):
        sm.smap_result_reduce(plan, small)
    with pytest.raises(TypeError):
        sm.smap_result_reduce(plan, np.zeros(7, np.int64))              # host buffer
    with pytest.raises(ValueError):
        sm.smap_result_combine(torch.zeros(7, dtype=torch.int64, device="cuda"), 2,
                               torch.zeros(7, dtype=torch.int64, device="cuda"))   # 2 records need 112 bytes


@pytest.mark.parametrize("m,n,kw,payload,param,flags_name,P", [
    (3, 1024, dict(rho=64, granularity="tile", persistent=32), "tc", 0.5, "none", 3),
    (3, 512, dict(rho=32, granularity="tile", layout="tiles"), "index_write_atm", 1e-2, "xor", 2),
    (3, 1024, dict(rho=64, granularity="tile", persistent=16, shard_rank=1, shard_count=4), "tc", 0.5, "none", 2),
])
def test_plans_in_flight_round_robin(sm, orc, m, n, kw, payload, param, flags_name, P):
    """Several steps in flight (`two_plans`): P plans of the same
    (shard of the) workload, their captured steps launched round robin on P streams
    with no ordering between consecutive steps; every plan's record equals the one
    of a plain smap_run, bit for bit (each plan owns its scratch, output and result
    block, so concurrent steps cannot interfere)."""
    flags = sm.RUN_XOR if flags_name == "xor" else 0
    p = workloads.points(n, 13)
    pts = torch.from_numpy(p).cuda()
    ref_plan = sm.smap_plan(m, n, **kw)
    ref_out = sm.alloc_out(ref_plan, payload)
    sm.smap_run(ref_plan, payload, points=pts, param=param, out=ref_out, flags=flags)
    ref = torch.zeros(7, dtype=torch.int64, device="cuda")
    sm.smap_result_reduce(ref_plan, ref)
    want = sm.result_dict(ref)
    streams = [torch.cuda.current_stream()] + [torch.cuda.Stream() for _ in range(P - 1)]
    gs = []
    for _ in range(P):
        plan = sm.smap_plan(m, n, **kw)
        out = sm.alloc_out(plan, payload)
        rec = torch.zeros(7, dtype=torch.int64, device="cuda")
        gs.append((plan, out, rec, sm.smap_graph_capture(plan, payload, points=pts, param=param, out=out,
                                                         flags=flags, record=rec)))
    torch.cuda.synchronize()
    for k in range(4 * P + 1):
        sm.smap_graph_launch(gs[k % P][3], stream=streams[k % P])
    torch.cuda.synchronize()
    for g in gs:
        assert sm.result_dict(g[2]) == want
    if payload == "tc" and "shard_count" not in kw:
        assert want["tc"] == orc.tc_count(p, np.float32(param))
