"""Multi-GPU host logic on CPU: the omega_x shard partition through
host-only plans of the C library, and the all-reduce of the per-rank result
records with world_size 2 over gloo (the bench uses NCCL with the same
record).  Each rank's record is what its GPU shard would produce; here it is
computed by the oracle over exactly the elements the shard owns."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

M64 = (1 << 64) - 1


def _mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z ^ (z >> np.uint64(30)); z = z * np.uint64(0xBF58476D1CE4E5B9)
        z = z ^ (z >> np.uint64(27)); z = z * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def shard_record(orc, m, inclusive, n, rho, rank, G):
    """(count, s0, s1, mix) of the index-write payload over the shard's elements."""
    hits, res = orc.element_hits(m, inclusive, False, n, rho, rank=rank, G=G)
    p = np.nonzero(hits)[0].astype(np.uint64)
    with np.errstate(over="ignore"):
        s0 = int(p.sum(dtype=np.uint64))
        s1 = int(((p + np.uint64(1)) * p).sum(dtype=np.uint64))
        mix = int(_mix64(p ^ (p * np.uint64(0x9E3779B97F4A7C15))).sum(dtype=np.uint64))
    return [len(p), s0, s1, mix]


def _to_i64(v):
    return [x - (1 << 64) if x >= (1 << 63) else x for x in v]


CASES = [(2, False, 512, 8, 2), (2, True, 256, 8, 2), (3, False, 128, 4, 2), (2, False, 256, 4, 4)]


@pytest.mark.parametrize("m,inc,n,rho,G", CASES)
def test_host_only_plans_partition_volume(m, inc, n, rho, G):
    import paper_1610_07394_b200 as sm
    diag = "inclusive" if inc else "strict"
    V = sm.smap_volume(m, n, diag)
    tot = 0
    blocks = set()
    for r in range(G):
        q = sm.smap_plan_query(sm.smap_plan(m, n, rho, diag=diag, shard_rank=r, shard_count=G,
                                            device=sm.DEVICE_NONE))
        tot += q["useful_elems"]
        blocks.add(q["grid_blocks"])
    assert tot == V and len(blocks) == 1
    plan = sm.smap_plan(m, n, rho, diag=diag, device=sm.DEVICE_NONE)
    with pytest.raises(sm.SmapError):
        sm.smap_run(plan, "index_write", out=0, out_bytes=0)


def test_shard_records_match_oracle_closed_form(orc):
    import paper_1610_07394_b200 as sm
    for m, inc, n, rho, G in CASES:
        recs = [shard_record(orc, m, inc, n, rho, r, G) for r in range(G)]
        for r in range(G):
            q = sm.smap_plan_query(sm.smap_plan(m, n, rho, diag="inclusive" if inc else "strict",
                                                shard_rank=r, shard_count=G, device=sm.DEVICE_NONE))
            assert recs[r][0] == q["useful_elems"]
        tot = [sum(x) & M64 for x in zip(*recs)]
        full = orc.cs_index(m, inc, n)
        assert tot == [full["count"], full["s0"], full["s1"], full["mix"]]


def _worker(rank, world, port, m, inc, n, rho, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_1610_07394_b200 as sm
    oracle.lib()
    plan = sm.smap_plan(m, n, rho, diag="inclusive" if inc else "strict", shard_rank=rank, shard_count=world,
                        device=sm.DEVICE_NONE)
    rec = shard_record(oracle, m, inc, n, rho, rank, world)
    t = torch.tensor(_to_i64(rec), dtype=torch.int64)
    dist.all_reduce(t)                                   # exact mod 2^64 (two's complement wrap)
    useful = torch.tensor([sm.smap_plan_query(plan)["useful_elems"]], dtype=torch.int64)
    allu = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allu, useful)
    if rank == 0:
        q.put(([int(x) & M64 for x in t.tolist()], [int(u) for u in allu]))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("m,inc,n,rho", [(2, False, 512, 8), (3, False, 128, 4)])
def test_gloo_world2_allreduce_of_shard_records(orc, m, inc, n, rho):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.start_processes(_worker, args=(2, _free_port(), m, inc, n, rho, q), nprocs=2, join=True, start_method="spawn")
    tot, useful = q.get()
    full = orc.cs_index(m, inc, n)
    assert tot == [full["count"], full["s0"], full["s1"], full["mix"]]
    assert useful[0] == useful[1] == full["count"] // 2     # exact volume balance


def _rec_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    rec = torch.tensor([100 + rank, -1, 5, 7, 0, 0x0F0F << rank, 0], dtype=torch.int64)
    rec[6:7] = torch.tensor([0.25 * (rank + 1)], dtype=torch.float64).view(torch.int64)
    g = torch.zeros(world * 7, dtype=torch.int64)
    dist.all_gather_into_tensor(g, rec)
    out = bench.combine_records(g.view(world, 7))
    if rank == 0:
        q.put(out.tolist())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_record_combine():
    """bench.py's a8 step: all-gather + combine of the 56-byte result records."""
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.start_processes(_rec_worker, args=(2, _free_port(), q), nprocs=2, join=True, start_method="spawn")
    out = q.get()
    assert out[0] == 201 and out[1] == -2 and out[2] == 10 and out[3] == 14
    assert out[5] == (0x0F0F ^ (0x0F0F << 1))
    assert torch.tensor(out[6:7], dtype=torch.int64).view(torch.float64).item() == 0.75
