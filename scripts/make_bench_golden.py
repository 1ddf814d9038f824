"""Write tests/golden/bench_expected.json: the oracle's results for the full
BASELINE workloads bench.py times, so that every bench run checks its timed
output against them.  Calls only oracle/ (plain C,
OpenMP over the host cores) and workloads.py (seeded inputs); no value comes
from the CUDA path.

    python scripts/make_bench_golden.py [--skip-c5x]

Fields per config: count and xr (xor of the 32/64-bit value patterns, the
bench's fused reduction E21') of the written outputs, for the index writes
also s0 (the sum of the values mod 2^64: xr of 0 .. V-1 is 0 for both index
configs, so the verification run uses RUN_CHECKSUM), the ATM sum (fp64,
compared at 1e-5 relative) and the TC count.  xr is independent of the output
layout and of the shard split (xor is associative), so one value serves the
tile-blocked layouts at every G.
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np

import oracle
import workloads

OUT = os.path.join(ROOT, "tests", "golden", "bench_expected.json")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-c5x", action="store_true", help="skip the n=8192 supplementary TC count")
    a = ap.parse_args()
    res = {"_source": "scripts/make_bench_golden.py (oracle/ only, workloads.py seeds)"}
    t = time.time()
    c = workloads.CONFIGS
    n = c["C2"]["n"]
    cs = oracle.cs_edm(workloads.points(n, workloads.SEED_C2))
    res["C2"] = {"n": n, "seed": workloads.SEED_C2, "payload": "edm", "count": cs["count"], "xr": cs["xr"]}
    print("C2", res["C2"], f"{time.time() - t:.1f}s", flush=True)
    n = c["C3"]["n"]
    cs = oracle.cs_index(3, False, n)
    p3 = workloads.points(n, workloads.SEED_C3)
    res["C3"] = {"n": n, "seed": workloads.SEED_C3, "payload": "index_write_atm", "count": cs["count"], "xr": cs["xr"],
                 "s0": cs["s0"],
                 "eps2": c["C3"]["eps2"], "atm_sum": oracle.atm_sum(p3, np.float32(c["C3"]["eps2"]))}
    print("C3", res["C3"], f"{time.time() - t:.1f}s", flush=True)
    n = c["C4"]["n"]
    cs = oracle.cs_index(2, False, n)
    res["C4"] = {"n": n, "payload": "index_write (u64)", "count": cs["count"], "xr": cs["xr"], "s0": cs["s0"]}
    print("C4", res["C4"], f"{time.time() - t:.1f}s", flush=True)
    n = c["C5"]["n"]
    p5 = workloads.points(n, workloads.SEED_C5)
    res["C5"] = {"n": n, "seed": workloads.SEED_C5, "payload": "tc", "R": c["C5"]["R"], "count": math.comb(n, 3),
                 "tc": oracle.tc_count(p5, np.float32(c["C5"]["R"]))}
    print("C5", res["C5"], f"{time.time() - t:.1f}s", flush=True)
    if not a.skip_c5x:
        n = workloads.C5X["n"]
        p = workloads.points(n, workloads.C5X["seed"])
        res["C5X"] = {"n": n, "seed": workloads.C5X["seed"], "payload": "tc", "R": workloads.C5X["R"],
                      "count": math.comb(n, 3), "tc": oracle.tc_count(p, np.float32(workloads.C5X["R"]))}
        print("C5X", res["C5X"], f"{time.time() - t:.1f}s", flush=True)
    elif os.path.exists(OUT):
        old = json.load(open(OUT))
        if "C5X" in old:
            res["C5X"] = old["C5X"]
    with open(OUT, "w") as f:
        json.dump(res, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
