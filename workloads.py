"""Seeded synthetic inputs and the BASELINE.json workload table.

A module of its own, shared by the oracle tests, the GPU parity tests and
bench.py.  It holds none of the method's arithmetic: only the random point
sets (uniform in [0,1)^3, fp32, n x 3 array-of-structs -- the point clouds of
the paper's n-body / EDM problem class) and the config
shapes.
"""
from __future__ import annotations

import numpy as np

# seeds per BASELINE.json config
SEED_C2 = 161007394
SEED_C3 = 161007395
SEED_C5 = 161007396

#: BASELINE.json configs -> concrete synthetic runs
CONFIGS = {
    "C1": dict(m=2, n=1024, rho=16, payload="index_write",
               desc="m=2, n=1024, block 16x16: lambda2 vs BB packed index write"),
    "C2": dict(m=2, n=65536, rho=16, payload="edm", seed=SEED_C2,
               desc="m=2 EDM lower triangle, n=65536 points in d=3 fp32, lambda2 vs BB on 1 B200"),
    "C3": dict(m=3, n=1024, rho=8, payload="index_write+atm", seed=SEED_C3, eps2=1e-2,
               desc="m=3, n=1024 tetrahedral index-write plus triple-interaction sum"),
    "C4": dict(m=2, n=1 << 17, rho=16, payload="index_write",
               desc="m=2 write-bound packed triangle, n=2^17, volume-sharded"),
    "C5": dict(m=3, n=2048, rho=8, payload="tc", seed=SEED_C5, R=0.5,
               desc="m=3 triple correlation over n=2048 random points, lambda3 sharded"),
}


#: supplementary C5 scaling workload ("a supplementary run with more
#: work as scaling evidence"): the same triple correlation at n = 8192 (64x the
#: triples of C5); not a BASELINE config, reported beside C5 only
SEED_C5X = 161007397
C5X = dict(m=3, n=8192, seed=SEED_C5X, R=0.5, desc="C5 at n=8192 (supplementary scaling run)")

#: launch configurations bench.py times (parity-tested at full size in
#: tests/test_gpu_fullsize.py).  Keys are smap_plan keyword arguments.
BENCH_EDM = dict(rho=256, granularity="tile", map="lambda", layout="tiles")
BENCH_EDM_VARIANTS = [BENCH_EDM, dict(rho=16, granularity="thread", map="lambda"),
                      dict(rho=256, granularity="tile", map="lambda"),
                      dict(rho=256, granularity="tile", map="bb", layout="tiles"),
                      dict(rho=128, granularity="tile", map="lambda", layout="tiles")]
BENCH_M3 = dict(rho=32, granularity="tile", map="lambda")
BENCH_M3_VARIANTS = [BENCH_M3, dict(rho=8, granularity="thread", map="lambda")]
BENCH_C3 = dict(rho=32, granularity="tile", map="lambda", layout="tiles")   # fused index write + ATM (E26)
BENCH_C4 = dict(rho=128, granularity="tile", map="lambda", layout="tiles")
# TC: 64-bit predicate rows; persistent >= 32 selects 64-thread CTAs (32 resident per SM).
# C5 (6144 tiles): one resident round of 32 CTAs/SM; C5X (n = 8192, 393K tiles): 256 per
# SM, i.e. 8 rounds the block scheduler hands out as CTAs finish -- dynamic balance over
# tiles of unequal cost (face tiles stage four bit tables), measured faster than one
# resident round at every G (profiles/r02_ab_tc_prepass_steps.log)
BENCH_C5 = dict(rho=64, granularity="tile", map="lambda", persistent=32)
BENCH_C5X = dict(rho=64, granularity="tile", map="lambda", persistent=256)


def sharded_launch(name: str, G: int) -> dict:
    """smap_plan keyword arguments of config `name`'s product launch on one of
    G omega_x shards (bench.py configs_sharded)."""
    base = {"C2": BENCH_EDM, "C3": BENCH_C3, "C4": BENCH_C4, "C5": BENCH_C5, "C5X": BENCH_C5X}[name]
    launch = dict(base)
    if name == "C5" and G > 1:
        # a shard has 6144 / G tiles: fewer than one per 64-thread CTA slot at G >= 2, where
        # 16 resident 128-thread CTAs per SM (half the k rows per thread) finish sooner
        launch["persistent"] = 16
    return launch


def points(n: int, seed: int) -> np.ndarray:
    """n x 3 fp32 points, uniform in [0,1)^3, from numpy's PCG64 stream."""
    return np.random.default_rng(seed).random((n, 3), dtype=np.float32)


def clustered_points(n: int, seed: int, copies: int = 4) -> np.ndarray:
    """Edge-case input: points with exact duplicates (zero distances)."""
    base = points((n + copies - 1) // copies, seed)
    return np.ascontiguousarray(np.repeat(base, copies, axis=0)[:n])
