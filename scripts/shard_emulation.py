"""Per-rank device time of the sharded launches, emulated on ONE GPU: every
rank r of G runs its omega_x column shard back to back;
the max over ranks is the kernel time a G-GPU run would see per step (the
collective -- one all-gather of 56 bytes -- comes on top).  Writes
gpurun_out/shards.json.

    python scripts/shard_emulation.py
"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1610_07394_b200 as sm
import workloads


def med(plan, payload, pts=None, param=0.0, out=None, flags=0, reps=8):
    for _ in range(2):
        sm.smap_run(plan, payload, points=pts, param=param, out=out, flags=flags)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        sm.smap_run(plan, payload, points=pts, param=param, out=out, flags=flags)
        b.record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in ev)
    return ts[len(ts) // 2]


def main():
    rows = []
    cases = [("C2 EDM", 2, workloads.CONFIGS["C2"]["n"], "edm", workloads.BENCH_EDM, workloads.SEED_C2, 0.0, sm.RUN_XOR),
             ("C3 IW+ATM", 3, workloads.CONFIGS["C3"]["n"], "index_write_atm", workloads.BENCH_C3, workloads.SEED_C3, 1e-2,
              sm.RUN_XOR),
             ("C4 IW u64", 2, workloads.CONFIGS["C4"]["n"], "index_write", workloads.BENCH_C4, None, 0.0, sm.RUN_XOR),
             ("C5 TC", 3, workloads.CONFIGS["C5"]["n"], "tc", workloads.BENCH_C5, workloads.SEED_C5, 0.5, 0)]
    for name, m, n, payload, cfg, seed, param, flags in cases:
        pts = torch.from_numpy(workloads.points(n, seed)).cuda() if seed else None
        row = {"config": name, "launch": cfg, "ranks": {}}
        for G in (1, 2, 4, 8):
            times = []
            for r in range(G):
                plan = sm.smap_plan(m, n, shard_rank=r, shard_count=G, **cfg)
                out = sm.alloc_out(plan, payload)
                times.append(med(plan, payload, pts, param, out, flags))
                st = sm.smap_stats_fetch(plan)
                del out
            torch.cuda.empty_cache()
            row["ranks"][G] = {"max_ms": round(max(times), 4), "min_ms": round(min(times), 4),
                               "speedup_vs_1": None}
        t1 = row["ranks"][1]["max_ms"]
        for G in (1, 2, 4, 8):
            row["ranks"][G]["speedup_vs_1"] = round(t1 / row["ranks"][G]["max_ms"], 3)
        print(json.dumps(row), flush=True)
        rows.append(row)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/shards.json", "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
