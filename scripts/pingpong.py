"""Step overlap across plans: the same shard's step captured on P plans (P pair
bitmaps / result blocks / outputs), launched round robin on P streams, so that
one step's pre-pass can overlap the previous step's count.  Compares the
per-step time of K back-to-back steps on one stream with the round robin.

    python scripts/pingpong.py --cfg C5X --G 8 --rank 0 [--plans 2]
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
    ap.add_argument("--cfg", default="C5X")
    ap.add_argument("--G", type=int, default=8)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--plans", type=int, default=2, help="plans (and streams) in flight")
    a = ap.parse_args()
    m, payload, seed, param = CASES[a.cfg]
    n = workloads.C5X["n"] if a.cfg == "C5X" else workloads.CONFIGS[a.cfg]["n"]
    pts = torch.from_numpy(workloads.points(n, seed)).cuda()
    launch = workloads.sharded_launch(a.cfg, a.G)
    flags = sm.RUN_XOR if payload == "index_write_atm" else 0
    graphs = []
    for _ in range(a.plans):
        plan = sm.smap_plan(m, n, shard_rank=a.rank, shard_count=a.G, **launch)
        out = sm.alloc_out(plan, payload)
        rec = torch.zeros(7, dtype=torch.int64, device="cuda")
        graphs.append((plan, out, rec, sm.smap_graph_capture(plan, payload, points=pts, param=param, out=out,
                                                             flags=flags, record=rec)))
    s0 = torch.cuda.current_stream()
    ss = [s0] + [torch.cuda.Stream() for _ in range(a.plans - 1)]
    one, two = [], []
    for _ in range(a.reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s0)
        for _ in range(a.steps):
            sm.smap_graph_launch(graphs[0][3], stream=s0)
        e1.record(s0)
        torch.cuda.synchronize()
        one.append(e0.elapsed_time(e1) / a.steps)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s0)
        for st in ss[1:]:
            st.wait_event(e0)
        for k in range(a.steps):
            sm.smap_graph_launch(graphs[k % a.plans][3], stream=ss[k % a.plans])
        for st in ss[1:]:
            d = torch.cuda.Event()
            d.record(st)
            s0.wait_event(d)
        e1.record(s0)
        torch.cuda.synchronize()
        two.append(e0.elapsed_time(e1) / a.steps)
    rs = [sm.result_dict(g[2]) for g in graphs]
    assert all(r == rs[0] for r in rs), rs
    r0 = rs[0]
    print(f"{a.cfg} G={a.G} rank={a.rank}: one stream {statistics.median(one[1:]) * 1e3:.1f} us/step, "
          f"{a.plans} plans round robin {statistics.median(two[1:]) * 1e3:.1f} us/step (tc={r0['tc']}, count={r0['count']})")


if __name__ == "__main__":
    main()
