"""One small run of every kernel family (for compute-sanitizer memcheck /
racecheck / synccheck on the GPU box):

    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1610_07394_b200 as sm
import workloads


def main():
    p2 = torch.from_numpy(workloads.points(1000, 1)).cuda()
    p3 = torch.from_numpy(workloads.points(300, 2)).cuda()
    runs = 0
    for mp in ("lambda", "bb", "below", "enum"):
        for gran, rho2, rho3 in (("thread", 16, 8), ("tile", 64, 16), ("tile", 128, 32)):
            if mp == "enum" and gran == "tile":
                continue
            for m, n, rho, pts in ((2, 1000, rho2, p2), (3, 300, rho3, p3)):
                for diag in ("strict", "inclusive"):
                    plan = sm.smap_plan(m, n, rho, map=mp, diag=diag, granularity=gran)
                    pls = ["index_write", "hitcount", "map_dump", "empty"]
                    if diag == "strict":
                        pls += ["edm"] if m == 2 else ["atm", "tc", "index_write_atm"]
                    for pl in pls:
                        out = sm.alloc_out(plan, pl, zero=True)
                        sm.smap_run(plan, pl, points=pts, param=0.5 if pl == "tc" else 1e-2, out=out,
                                    flags=sm.RUN_CHECKSUM_MIX if pl in ("index_write", "edm", "index_write_atm") else 0)
                        sm.smap_stats_fetch(plan)
                        runs += 1
    # the E29 tile layout of below plans (any n, holes), incl. the fused payload
    for m, n, rho, pl in ((2, 1000, 64, "edm"), (2, 1000, 128, "index_write"), (3, 300, 32, "index_write_atm"),
                          (3, 300, 16, "index_write")):
        pts = torch.from_numpy(workloads.points(n, 4)).cuda()
        plan = sm.smap_plan(m, n, rho, map="below", granularity="tile", layout="tiles")
        out = sm.alloc_out(plan, pl)
        sm.smap_run(plan, pl, points=pts, param=1e-2, out=out, flags=sm.RUN_CHECKSUM_MIX)
        sm.smap_stats_fetch(plan)
        runs += 1
    # tile layouts, sharded
    for m, n, rho in ((2, 1024, 64), (3, 256, 16), (3, 256, 32)):
        pts = torch.from_numpy(workloads.points(n, 3)).cuda()
        for r in range(2):
            plan = sm.smap_plan(m, n, rho, granularity="tile", layout="tiles", shard_rank=r, shard_count=2)
            for pl in ("index_write",) + (("edm",) if m == 2 else ("index_write_atm",)):
                out = sm.alloc_out(plan, pl)
                sm.smap_run(plan, pl, points=pts, param=1e-2, out=out, flags=sm.RUN_XOR)
                sm.smap_stats_fetch(plan)
                runs += 1
    # the benchmarked EDM launches (VEC 16-B stores, warp-private staging reused across
    # persistent tiles) with the timed step's reductions, plus the smap_run_host path
    for n, rho, persistent in ((1024, 256, 0), (8192, 256, 1), (1024, 128, 0), (8192, 128, 1), (1000, 256, 0)):
        pts = torch.from_numpy(workloads.points(n, 5)).cuda()
        mp = "below" if n % rho else "lambda"
        plan = sm.smap_plan(2, n, rho, map=mp, granularity="tile", layout="tiles", persistent=persistent)
        out = sm.alloc_out(plan, "edm")
        for flags in (sm.RUN_XOR, sm.RUN_CHECKSUM, 0):
            sm.smap_run(plan, "edm", points=pts, out=out, flags=flags)
            sm.smap_stats_fetch(plan)
            runs += 1
        sm.smap_run_host(plan, "edm", host_points=workloads.points(n, 5), out=out, flags=sm.RUN_XOR)
        runs += 1
    # the benchmarked C3 / C4 / C5 launches at reduced n
    p3 = torch.from_numpy(workloads.points(512, 6)).cuda()
    for kw, pl, n, param in ((workloads.BENCH_C3, "index_write_atm", 512, 1e-2), (workloads.BENCH_C4, "index_write", 2048, 0.0),
                             (workloads.BENCH_C5, "tc", 512, 0.5)):
        plan = sm.smap_plan(2 if pl == "index_write" else 3, n, **kw)
        out = sm.alloc_out(plan, pl)
        sm.smap_run(plan, pl, points=p3 if pl != "index_write" else None, param=param, out=out,
                    flags=sm.RUN_XOR if pl != "tc" else 0)
        sm.smap_stats_fetch(plan)
        runs += 1
    # round 2: SMAP_RUN_FAST_SQRT (incl. the staging fallback), the symmetric TC pre-pass at
    # T = 64 with a padded n, and lean CUDA-graph steps (record folded into the finalize,
    # programmatic-dependent tail kernels, result block cleared behind the record)
    for scale in (1.0, 1e-15):
        pts = torch.from_numpy((workloads.points(1024, 7) * scale).astype("float32")).cuda()
        plan = sm.smap_plan(2, 1024, 256, granularity="tile", layout="tiles")
        out = sm.alloc_out(plan, "edm")
        sm.smap_run(plan, "edm", points=pts, out=out, flags=sm.RUN_XOR | sm.RUN_FAST_SQRT)
        sm.smap_stats_fetch(plan)
        runs += 1
    for n in (1000, 1024):
        pts = torch.from_numpy(workloads.points(n, 8)).cuda()
        plan = sm.smap_plan(3, n, 64, granularity="tile", persistent=8)
        sm.smap_run(plan, "tc", points=pts, param=0.5)
        sm.smap_stats_fetch(plan)
        runs += 1
    # round 2 (late): the rewritten pair-bitmap pre-pass (blocked layout, warp bit transpose)
    # unsharded and with the shard block lists, T = 32 / 64, all three TC CTA sizes, padded n
    for n, rho, persistent, G in ((1000, 64, 32, 1), (1000, 64, 16, 3), (1000, 32, 0, 2), (777, 64, 256, 2)):
        pts = torch.from_numpy(workloads.points(n, 10)).cuda()
        for r in range(G):
            plan = sm.smap_plan(3, n, rho, granularity="tile", persistent=persistent, shard_rank=r, shard_count=G)
            sm.smap_run(plan, "tc", points=pts, param=0.5)
            sm.smap_stats_fetch(plan)
            runs += 1
    rec = torch.zeros(7, dtype=torch.int64, device="cuda")
    for m, n, kw, pl in ((3, 512, workloads.BENCH_C3, "index_write_atm"), (3, 512, workloads.BENCH_M3, "atm"),
                         (3, 1024, workloads.BENCH_C5, "tc"), (2, 2048, workloads.BENCH_C4, "index_write")):
        pts = torch.from_numpy(workloads.points(n, 9)).cuda() if pl != "index_write" else None
        plan = sm.smap_plan(m, n, **kw)
        out = sm.alloc_out(plan, pl)
        g = sm.smap_graph_capture(plan, pl, points=pts, param=0.5 if pl == "tc" else 1e-2, out=out,
                                  flags=sm.RUN_XOR if pl in ("index_write", "index_write_atm") else 0, record=rec)
        for _ in range(2):
            sm.smap_graph_launch(g)
            runs += 1
        sm.smap_run(plan, pl, points=pts, param=0.5 if pl == "tc" else 1e-2, out=out)   # leaves the block dirty
        sm.smap_graph_launch(g)
        runs += 2
    torch.cuda.synchronize()
    print(f"sanitize cases: {runs} runs ok")


if __name__ == "__main__":
    main()
