"""Quick device-time survey of the kernels (CUDA events, median of reps).
Not the bench: prints one line per configuration for exploration."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1610_07394_b200 as sm
import workloads


def time_run(plan, payload, pts=None, param=0.0, out=None, flags=0, reps=10, warm=3):
    s = torch.cuda.current_stream()
    for _ in range(warm):
        sm.smap_run(plan, payload, points=pts, param=param, out=out, flags=flags)
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(reps)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(reps)]
    for k in range(reps):
        e0[k].record(s)
        sm.smap_run(plan, payload, points=pts, param=param, out=out, flags=flags)
        e1[k].record(s)
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in zip(e0, e1))
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="all")
    args = ap.parse_args()
    rows = []
    dev = torch.cuda.get_device_properties(0)
    print(f"# {dev.name} SMs={dev.multi_processor_count}", flush=True)

    def rec(name, m, n, cfg, payload, ms, V, bytes_per=0):
        r = dict(name=name, m=m, n=n, cfg=cfg, payload=payload, ms=round(ms, 4), elems_per_s=V / (ms * 1e-3),
                 gbs=(V * bytes_per / (ms * 1e-3) / 1e9) if bytes_per else None)
        rows.append(r)
        print(json.dumps(r), flush=True)

    if args.which in ("all", "edm"):
        n = 65536
        p = torch.from_numpy(workloads.points(n, workloads.SEED_C2)).cuda()
        V = n * (n - 1) // 2
        out = torch.empty(V, dtype=torch.float32, device="cuda")
        for cfg in [dict(rho=128, granularity="tile"), dict(rho=128, granularity="tile", order="squares"),
                    dict(rho=256, granularity="tile"), dict(rho=256, granularity="tile", order="squares"),
                    dict(rho=512, granularity="tile"), dict(rho=512, granularity="tile", order="squares"),
                    dict(rho=256, granularity="tile", persistent=4),
                    dict(rho=512, granularity="tile", persistent=4)]:
            for mp in ("lambda", "bb"):
                if mp == "bb" and cfg.get("order") == "squares":
                    continue
                plan = sm.smap_plan(2, n, map=mp, **cfg)
                for flags in (0, 1):
                    ms = time_run(plan, "edm", pts=p, out=out, flags=flags)
                    rec(f"edm-{mp}-cs{flags}", 2, n, cfg, "edm", ms, V, 4)
        del out
        torch.cuda.empty_cache()
    if args.which in ("all", "iw2"):
        n = 65536
        V = n * (n - 1) // 2
        out = torch.empty(V, dtype=torch.int32, device="cuda")
        for cfg in [dict(rho=16, granularity="thread"), dict(rho=128, granularity="tile", persistent=4),
                    dict(rho=128, granularity="tile")]:
            for mp in ("lambda", "bb"):
                plan = sm.smap_plan(2, n, map=mp, **cfg)
                ms = time_run(plan, "index_write", out=out)
                rec(f"iw2-{mp}", 2, n, cfg, "index_write", ms, V, 4)
                ms = time_run(plan, "empty")
                rec(f"empty2-{mp}", 2, n, cfg, "empty", ms, V)
        del out
        torch.cuda.empty_cache()
    if args.which in ("all", "m3"):
        n = 1024
        V = n * (n - 1) * (n - 2) // 6
        p = torch.from_numpy(workloads.points(n, workloads.SEED_C3)).cuda()
        out = torch.empty(V, dtype=torch.int32, device="cuda")
        for cfg in [dict(rho=8, granularity="thread"), dict(rho=16, granularity="tile"), dict(rho=32, granularity="tile"),
                    dict(rho=32, granularity="tile", persistent=4), dict(rho=16, granularity="tile", persistent=8)]:
            for mp in ("lambda", "bb"):
                plan = sm.smap_plan(3, n, map=mp, **cfg)
                ms = time_run(plan, "index_write", out=out)
                rec(f"iw3-{mp}", 3, n, cfg, "index_write", ms, V, 4)
                ms = time_run(plan, "atm", pts=p, param=1e-2)
                rec(f"atm-{mp}", 3, n, cfg, "atm", ms, V)
                ms = time_run(plan, "empty")
                rec(f"empty3-{mp}", 3, n, cfg, "empty", ms, V)
        n = 2048
        V = n * (n - 1) * (n - 2) // 6
        p = torch.from_numpy(workloads.points(n, workloads.SEED_C5)).cuda()
        for cfg in [dict(rho=8, granularity="thread"), dict(rho=32, granularity="tile", persistent=4),
                    dict(rho=16, granularity="tile", persistent=8)]:
            for mp in ("lambda", "bb"):
                plan = sm.smap_plan(3, n, map=mp, **cfg)
                ms = time_run(plan, "tc", pts=p, param=0.5)
                rec(f"tc-{mp}", 3, n, cfg, "tc", ms, V)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/explore.json", "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
