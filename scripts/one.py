"""Run one configuration a few times (for ncu captures and quick timing).

  python scripts/one.py --m 2 --n 65536 --payload edm --rho 128 --gran tile --map lambda --reps 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1610_07394_b200 as sm
import workloads


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=2)
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--payload", default="edm")
    ap.add_argument("--rho", type=int, default=128)
    ap.add_argument("--gran", default="tile")
    ap.add_argument("--map", default="lambda")
    ap.add_argument("--persistent", type=int, default=0)
    ap.add_argument("--layout", default="rows")
    ap.add_argument("--order", default="rows")
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--param", type=float, default=0.5)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--memset", action="store_true", help="also time a cudaMemset of the output (write roofline)")
    a = ap.parse_args()
    plan = sm.smap_plan(a.m, a.n, a.rho, map=a.map, granularity=a.gran, persistent=a.persistent,
                        layout=a.layout, order=a.order)
    pts = torch.from_numpy(workloads.points(a.n, 7)).cuda()
    out = sm.alloc_out(plan, a.payload)
    for _ in range(a.reps):
        sm.smap_run(plan, a.payload, points=pts, param=a.param, out=out, flags=a.flags)
        st = sm.smap_stats_fetch(plan)
        print(f"{a.payload} {a.map} {a.gran} rho={a.rho} p={a.persistent}: {st['kernel_ms']:.4f} ms count={st['count']}")
    if a.memset and out is not None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(3):
            e0.record(); out.zero_(); e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            nb = out.numel() * out.element_size()
            print(f"fill {nb/1e9:.2f} GB: {ms:.4f} ms = {nb/ms/1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
