"""Relative error of the GPU ATM sum against the oracle's fp64-accumulated
fp32 terms (tolerance 1e-5, north_star), for every ATM kernel path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import oracle
import paper_1610_07394_b200 as sm
import workloads

for n, eps2 in [(256, 1e-2), (256, 0.0), (333, 1e-2), (1024, 1e-2), (1024, 0.0)]:
    p = workloads.points(n, workloads.SEED_C3)
    ref = oracle.atm_sum(p, np.float32(eps2))
    dp = torch.from_numpy(p).cuda()
    for cfg in (dict(rho=32, granularity="tile"), dict(rho=16, granularity="tile"), dict(rho=8, granularity="thread")):
        for mp in ("lambda", "bb"):
            plan = sm.smap_plan(3, n, map=mp, **cfg)
            sm.smap_run(plan, "atm", points=dp, param=eps2)
            st = sm.smap_stats_fetch(plan)
            print(f"n={n} eps2={eps2} {mp} {cfg['granularity']} rho={cfg['rho']}: rel err {abs(st['sum'] - ref) / abs(ref):.2e}")
