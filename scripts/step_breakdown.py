"""Where a sharded step's time goes: one rank's CUDA-graph step timed alone
(events around one launch, as shard_emulation.py does), pipelined (many
launches between two events: no host submission gap), and -- under
`ncu --metrics gpu__time_duration.sum` -- each kernel of the step.

    python scripts/step_breakdown.py --cfg C3 --G 8 --rank 0
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1610_07394_b200 as sm
import workloads

CASES = {"C3": (3, "index_write_atm", workloads.SEED_C3, 1e-2), "C5": (3, "tc", workloads.SEED_C5, 0.5),
         "C5X": (3, "tc", workloads.SEED_C5X, 0.5)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="C3")
    ap.add_argument("--G", type=int, default=8)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--rho", type=int, default=0)
    ap.add_argument("--persistent", type=int, default=-1)
    a = ap.parse_args()
    m, payload, seed, param = CASES[a.cfg]
    n = workloads.C5X["n"] if a.cfg == "C5X" else workloads.CONFIGS[a.cfg]["n"]
    pts = torch.from_numpy(workloads.points(n, seed)).cuda()
    launch = workloads.sharded_launch(a.cfg, a.G)
    if a.rho:
        launch["rho"] = a.rho
    if a.persistent >= 0:
        launch["persistent"] = a.persistent
    flags = sm.RUN_XOR if payload == "index_write_atm" else 0
    plan = sm.smap_plan(m, n, shard_rank=a.rank, shard_count=a.G, **launch)
    out = sm.alloc_out(plan, payload)
    rec = torch.zeros(7, dtype=torch.int64, device="cuda")
    g = sm.smap_graph_capture(plan, payload, points=pts, param=param, out=out, flags=flags, record=rec)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    alone, piped = [], []
    for rep in range(a.reps):
        e0.record(); sm.smap_graph_launch(g); e1.record(); torch.cuda.synchronize()
        alone.append(e0.elapsed_time(e1))
        e0.record()
        for _ in range(10):
            sm.smap_graph_launch(g)
        e1.record(); torch.cuda.synchronize()
        piped.append(e0.elapsed_time(e1) / 10)
    r = sm.result_dict(rec)
    print(f"{a.cfg} G={a.G} rank={a.rank} {launch}: alone {statistics.median(alone)*1e3:.1f} us, "
          f"pipelined {statistics.median(piped)*1e3:.1f} us per step; count={r['count']} tc={r['tc']}")


if __name__ == "__main__":
    main()
