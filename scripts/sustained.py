"""Sustained vs burst behaviour under the board power cap: K back-to-back
launches of each selected kernel on the C2 output buffer (8.59 GB), with
per-launch CUDA-event times and nvidia-smi clocks / power sampled alongside.

  edm   the C2 EDM kernel (bench launch, count + xor reduction)
  iw    the m=2 u32 index write with the same launch and the same 8.59 GB
        (SM stores with almost no arithmetic: separates store-path power
        from EDM arithmetic power)
  fill  torch's write fill of the same buffer (the write roofline)

Writes gpurun_out/sustained[_TAG].json and prints one summary line per kernel.

    python scripts/sustained.py [--k 400] [--what edm,iw,fill] [--tag base]
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
    ap.add_argument("--what", default="edm,fill")
    ap.add_argument("--tag", default="")
    ap.add_argument("--cool", type=float, default=2.0, help="idle seconds before each kernel's run")
    a = ap.parse_args()
    n = 65536
    pts = torch.from_numpy(workloads.points(n, workloads.SEED_C2)).cuda()
    plan = sm.smap_plan(2, n, **workloads.BENCH_EDM)
    out = sm.alloc_out(plan, "edm")
    outi = out.view(torch.int32)
    rows, stop = [], threading.Event()
    th = threading.Thread(target=sampler, args=(rows, stop), daemon=True)
    th.start()
    time.sleep(1.0)
    fns = {"edm": lambda: sm.smap_run(plan, "edm", points=pts, out=out, flags=sm.RUN_XOR),
           "iw": lambda: sm.smap_run(plan, "index_write", out=outi, flags=sm.RUN_XOR),
           "fill": lambda: out.zero_()}
    res = {}
    for name in a.what.split(","):
        time.sleep(a.cool)                                 # let the board cool down between kernels
        t0 = time.perf_counter()
        ts = run(fns[name], a.k)
        t1 = time.perf_counter()
        smp = [r for t, r in rows if t0 <= t <= t1]
        tail = [r for t, r in rows if t0 + 0.5 * (t1 - t0) <= t <= t1]
        sm_mhz = [float(r.split(",")[0]) for r in tail if r.split(",")[0].strip().replace(".", "").isdigit()]
        pw = [float(r.split(",")[2]) for r in tail if r.split(",")[2].strip().replace(".", "").isdigit()]
        res[name] = {"first10_ms": [round(x, 4) for x in ts[:10]], "median_first50": statistics.median(ts[:50]),
                     "median_last100": statistics.median(ts[-100:]), "samples": smp[::max(1, len(smp) // 12)],
                     "sm_mhz_median_2nd_half": statistics.median(sm_mhz) if sm_mhz else None,
                     "power_w_median_2nd_half": statistics.median(pw) if pw else None}
    stop.set()
    nb = out.numel() * 4
    for k in res:
        res[k]["gbs_first50"] = nb / res[k]["median_first50"] / 1e6
        res[k]["gbs_last100"] = nb / res[k]["median_last100"] / 1e6
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/sustained{'_' + a.tag if a.tag else ''}.json", "w") as f:
        json.dump(res, f, indent=1)
    for k, v in res.items():
        print(f"{a.tag or '-'} {k}: burst {v['gbs_first50']:.0f} GB/s, last100 {v['gbs_last100']:.0f} GB/s "
              f"({v['median_last100']:.4f} ms), sm {v['sm_mhz_median_2nd_half']} MHz, {v['power_w_median_2nd_half']} W")


if __name__ == "__main__":
    main()
