"""Sustained vs burst behaviour under the board power cap: K back-to-back
launches of the C2 EDM kernel, then K back-to-back write fills of the same
buffer, per-launch CUDA-event times with nvidia-smi clocks / power sampled
alongside.  Writes gpurun_out/sustained.json.

    python scripts/sustained.py [--k 400]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1610_07394_b200 as sm
import workloads


def sampler(rows, stop):
    p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,clocks.mem,power.draw,clocks_event_reasons.sw_power_cap",
                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
    for line in p.stdout:
        rows.append((time.perf_counter(), line.strip()))
        if stop.is_set():
            break
    p.terminate()


def run(fn, k):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=400)
    a = ap.parse_args()
    n = 65536
    pts = torch.from_numpy(workloads.points(n, workloads.SEED_C2)).cuda()
    plan = sm.smap_plan(2, n, **workloads.BENCH_EDM)
    out = sm.alloc_out(plan, "edm")
    rows, stop = [], threading.Event()
    th = threading.Thread(target=sampler, args=(rows, stop), daemon=True)
    th.start()
    time.sleep(1.0)
    res = {}
    for name, fn in (("edm", lambda: sm.smap_run(plan, "edm", points=pts, out=out, flags=sm.RUN_XOR)),
                     ("fill", lambda: out.zero_())):
        time.sleep(1.0)                                   # let the board cool down between the two
        t0 = time.perf_counter()
        ts = run(fn, a.k)
        t1 = time.perf_counter()
        smp = [r for t, r in rows if t0 <= t <= t1]
        res[name] = {"first10_ms": [round(x, 4) for x in ts[:10]], "median_first50": statistics.median(ts[:50]),
                     "median_last100": statistics.median(ts[-100:]), "samples": smp[::max(1, len(smp) // 12)]}
    stop.set()
    nb = out.numel() * 4
    for k in res:
        res[k]["gbs_first50"] = nb / res[k]["median_first50"] / 1e6
        res[k]["gbs_last100"] = nb / res[k]["median_last100"] / 1e6
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/sustained.json", "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: {x: v[x] for x in ("median_first50", "median_last100", "gbs_first50", "gbs_last100")} for k, v in res.items()}, indent=1))
    for k in res:
        print(k, res[k]["samples"])


if __name__ == "__main__":
    main()
