"""Step overlap across two plans: the same shard's step captured twice (two
plans = two pair bitmaps / result blocks), launched alternately on two streams,
so that one step's pre-pass can overlap the previous step's count.  Compares
the per-step time of K back-to-back steps on one stream with the ping-pong.

    python scripts/pingpong.py --cfg C5X --G 8 --rank 0
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
    a = ap.parse_args()
    m, payload, seed, param = CASES[a.cfg]
    n = workloads.C5X["n"] if a.cfg == "C5X" else workloads.CONFIGS[a.cfg]["n"]
    pts = torch.from_numpy(workloads.points(n, seed)).cuda()
    launch = workloads.sharded_launch(a.cfg, a.G)
    flags = sm.RUN_XOR if payload == "index_write_atm" else 0
    graphs = []
    for _ in range(2):
        plan = sm.smap_plan(m, n, shard_rank=a.rank, shard_count=a.G, **launch)
        out = sm.alloc_out(plan, payload)
        rec = torch.zeros(7, dtype=torch.int64, device="cuda")
        graphs.append((plan, out, rec, sm.smap_graph_capture(plan, payload, points=pts, param=param, out=out,
                                                             flags=flags, record=rec)))
    s0 = torch.cuda.current_stream()
    s1 = torch.cuda.Stream()
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
        s1.wait_event(e0)
        for k in range(a.steps):
            sm.smap_graph_launch(graphs[k % 2][3], stream=s0 if k % 2 == 0 else s1)
        done1 = torch.cuda.Event()
        done1.record(s1)
        s0.wait_event(done1)
        e1.record(s0)
        torch.cuda.synchronize()
        two.append(e0.elapsed_time(e1) / a.steps)
    r0, r1 = sm.result_dict(graphs[0][2]), sm.result_dict(graphs[1][2])
    assert r0 == r1, (r0, r1)
    print(f"{a.cfg} G={a.G} rank={a.rank}: one stream {statistics.median(one[1:]) * 1e3:.1f} us/step, "
          f"two plans ping-pong {statistics.median(two[1:]) * 1e3:.1f} us/step (tc={r0['tc']}, count={r0['count']})")


if __name__ == "__main__":
    main()
