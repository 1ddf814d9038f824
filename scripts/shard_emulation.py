"""Per-rank device time of the sharded launches, emulated on ONE GPU: every
rank r of G runs its omega_x column shard as bench.py's
configs_sharded does -- one CUDA graph per rank step (payload kernels + the
record reduction, smap_graph_capture) -- and the max over ranks is the step
time a G-GPU run would see (the collective, one all-gather of 56 bytes, comes
on top).  Ranks are timed interleaved, in both orders, so that clock and
power drift hit every rank alike.  Writes gpurun_out/shards.json.

    python scripts/shard_emulation.py [--only C5,C5X] [--reps 9]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1610_07394_b200 as sm
import workloads

PIPE = 8   # steps per pipelined sample
TWO_PLANS = ("C3", "C5", "C5X")   # also timed with two plans in flight (the m=3 jobs with fixed step costs)

CASES = {"C2": (2, "edm", workloads.SEED_C2, 0.0), "C3": (3, "index_write_atm", workloads.SEED_C3, 1e-2),
         "C4": (2, "index_write", None, 0.0), "C5": (3, "tc", workloads.SEED_C5, 0.5),
         "C5X": (3, "tc", workloads.SEED_C5X, 0.5)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C2,C3,C4,C5,C5X")
    ap.add_argument("--reps", type=int, default=9)
    ap.add_argument("--gs", default="1,2,4,8")
    a = ap.parse_args()
    rows = []
    for name in a.only.split(","):
        m, payload, seed, param = CASES[name]
        n = workloads.C5X["n"] if name == "C5X" else workloads.CONFIGS[name]["n"]
        pts = torch.from_numpy(workloads.points(n, seed)).cuda() if seed else None
        flags = sm.RUN_XOR if payload in ("edm", "index_write", "index_write_atm") else 0
        row = {"config": name, "n": n, "payload": payload, "ranks": {}}
        for G in (int(g) for g in a.gs.split(",")):
            launch = workloads.sharded_launch(name, G)
            ranks = []
            two = name in TWO_PLANS
            for r in range(G):
                plan = sm.smap_plan(m, n, shard_rank=r, shard_count=G, **launch)
                out = sm.alloc_out(plan, payload)
                rec = torch.zeros(7, dtype=torch.int64, device="cuda")
                g = sm.smap_graph_capture(plan, payload, points=pts, param=param, out=out, flags=flags, record=rec)
                g2 = None
                if two:     # a second plan of the same shard (own scratch / output) for two steps in flight
                    plan2 = sm.smap_plan(m, n, shard_rank=r, shard_count=G, **launch)
                    out2 = sm.alloc_out(plan2, payload)
                    rec2 = torch.zeros(7, dtype=torch.int64, device="cuda")
                    g2 = (plan2, out2, rec2, sm.smap_graph_capture(plan2, payload, points=pts, param=param, out=out2,
                                                                   flags=flags, record=rec2))
                ranks.append((plan, out, rec, g, g2))
                if name == "C4" and G == 1:
                    break
            times = [[] for _ in ranks]
            piped = [[] for _ in ranks]
            twop = [[] for _ in ranks]
            s1 = torch.cuda.Stream()
            for rep in range(a.reps + 2):
                order = list(range(len(ranks))) if rep % 2 == 0 else list(reversed(range(len(ranks))))
                for r in order:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    sm.smap_graph_launch(ranks[r][3])
                    e1.record()
                    torch.cuda.synchronize()
                    if rep >= 2:
                        times[r].append(e0.elapsed_time(e1))
                    # the same rank's step PIPELINED (PIPE launches back to back between two
                    # events, as bench.py enqueues its timed steps): no host submission gap
                    e0.record()
                    for _ in range(PIPE):
                        sm.smap_graph_launch(ranks[r][3])
                    e1.record()
                    torch.cuda.synchronize()
                    if rep >= 2:
                        piped[r].append(e0.elapsed_time(e1) / PIPE)
                    if ranks[r][4] is not None:
                        # two plans alternating over two streams (step k+1 overlaps step k's tail)
                        s0 = torch.cuda.current_stream()
                        e0.record()
                        s1.wait_event(e0)
                        for k in range(PIPE):
                            sm.smap_graph_launch(ranks[r][3] if k % 2 == 0 else ranks[r][4][3],
                                                 stream=s0 if k % 2 == 0 else s1)
                        j = torch.cuda.Event()
                        j.record(s1)
                        s0.wait_event(j)
                        e1.record()
                        torch.cuda.synchronize()
                        if rep >= 2:
                            twop[r].append(e0.elapsed_time(e1) / PIPE)
            med = [statistics.median(t) for t in times]
            medp = [statistics.median(t) for t in piped]
            tot = {k: sum(sm.result_dict(x[2])[k] for x in ranks) for k in ("count", "tc")}
            for x in ranks:                 # the second plan's steps produced the same record
                if x[4] is not None:
                    assert sm.result_dict(x[4][2]) == sm.result_dict(x[2]), name
            medt = [statistics.median(t) for t in twop] if twop[0] else None
            row["ranks"][G] = {"launch": launch, "max_ms": round(max(med), 4), "min_ms": round(min(med), 4),
                               "max_ms_two_plans": round(max(medt), 4) if medt else None,
                               "per_rank_ms": [round(x, 4) for x in med],
                               "max_ms_pipelined": round(max(medp), 4), "min_ms_pipelined": round(min(medp), 4),
                               "per_rank_ms_pipelined": [round(x, 4) for x in medp],
                               "count": tot["count"], "tc": tot["tc"]}
            del ranks
            torch.cuda.empty_cache()
        t1 = row["ranks"][min(row["ranks"])]["max_ms"]
        t1p = row["ranks"][min(row["ranks"])]["max_ms_pipelined"]
        for G in row["ranks"]:
            v = row["ranks"][G]
            v["speedup_vs_1"] = round(t1 / v["max_ms"], 3)
            v["max_over_min"] = round(v["max_ms"] / v["min_ms"], 3)
            v["speedup_vs_1_pipelined"] = round(t1p / v["max_ms_pipelined"], 3)
            t1t = row["ranks"][min(row["ranks"])]["max_ms_two_plans"]
            if t1t:
                v["speedup_vs_1_two_plans"] = round(t1t / v["max_ms_two_plans"], 3)
        print(json.dumps({"config": name, **{G: (v["max_ms"], v["speedup_vs_1"], v["max_over_min"],
                                                 v["max_ms_pipelined"], v["speedup_vs_1_pipelined"],
                                                 v["max_ms_two_plans"], v.get("speedup_vs_1_two_plans"))
                                              for G, v in row["ranks"].items()}}), flush=True)
        rows.append(row)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/shards.json", "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
