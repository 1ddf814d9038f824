"""Device-time table of every BASELINE.json config (C1..C5): lambda vs BB at the
paper's one-element-per-thread granularity and at tile granularity, plus the
root-based enumeration map (SMAP_MAP_ENUM) at thread granularity.
CUDA events on the launching stream, warm-up, median of reps.  Writes
gpurun_out/configs.json (copied into profiles/ per round).

    python scripts/configs_bench.py [--only C2,C5] [--reps 10]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

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


def compare(m, n, payload, variants, pts=None, param=0.0, out=None, reps=10, diag="strict"):
    rows = []
    for name, cfg in variants:
        res = {"variant": name, "cfg": cfg}
        maps = ("lambda", "bb") + (("enum",) if cfg.get("granularity") == "thread" else ())
        for mp in maps:
            c = dict(cfg)
            flags = c.pop("flags", 0)
            if mp != "lambda":
                c.pop("order", None)
            plan = sm.smap_plan(m, n, map=mp, diag=diag, **c)
            q = sm.smap_plan_query(plan)
            ms = time_run(plan, payload, pts=pts, param=param, out=out, reps=reps, flags=flags)
            res[mp] = {"ms": round(ms, 4), "launched": q["launched_threads"], "blocks": q["grid_blocks"]}
            ems = time_run(plan, "empty", reps=reps)
            res[mp]["empty_ms"] = round(ems, 4)
            del plan
        V = sm.smap_volume(m, n, diag)
        res["elements"] = V
        res["lambda_elems_per_s"] = V / (res["lambda"]["ms"] * 1e-3)
        res["speedup_lambda_vs_bb"] = round(res["bb"]["ms"] / res["lambda"]["ms"], 3)
        res["launch_ratio_bb_over_lambda"] = round(res["bb"]["launched"] / res["lambda"]["launched"], 4)
        if "enum" in res:       # root-based enumeration map: same payload, fewer blocks than lambda3
            res["speedup_lambda_vs_enum"] = round(res["enum"]["ms"] / res["lambda"]["ms"], 3)
        print(json.dumps(res), flush=True)
        rows.append(res)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C1,C2,C3,C4,C5")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    only = set(a.only.split(","))
    dev = torch.cuda.get_device_properties(0)
    table = {"device": dev.name, "sms": dev.multi_processor_count, "configs": {}}
    thread2 = ("thread_rho16", dict(rho=16, granularity="thread"))
    thread2b = ("thread_rho32", dict(rho=32, granularity="thread"))
    if "C1" in only:
        n = 1024
        out = torch.empty(sm.smap_volume(2, n, "inclusive"), dtype=torch.int32, device="cuda")
        rows = compare(2, n, "index_write", [thread2, ("tile_rho128", dict(rho=128, granularity="tile"))],
                       out=out, reps=a.reps)
        rows += compare(2, n, "index_write", [thread2], out=out, reps=a.reps, diag="inclusive")
        table["configs"]["C1"] = rows
    if "C2" in only:
        n = 65536
        p = torch.from_numpy(workloads.points(n, workloads.SEED_C2)).cuda()
        out = torch.empty(sm.smap_volume(2, n), dtype=torch.float32, device="cuda")
        T = dict(granularity="tile", layout="tiles")
        table["configs"]["C2"] = compare(2, n, "edm", [thread2, thread2b, ("tile_rho256_rows", dict(rho=256, granularity="tile")),
                                                        ("tile_rho128_tiles", dict(rho=128, **T)),
                                                        ("tile_rho128_tiles_xor", dict(rho=128, flags=sm.RUN_XOR, **T)),
                                                        ("tile_rho128_tiles_p4_xor", dict(rho=128, persistent=4, flags=sm.RUN_XOR, **T)),
                                                        ("tile_rho128_tiles_p8_xor", dict(rho=128, persistent=8, flags=sm.RUN_XOR, **T)),
                                                        ("tile_rho256_tiles_xor", dict(rho=256, flags=sm.RUN_XOR, **T)),
                                                        ("tile_rho64_tiles_xor", dict(rho=64, flags=sm.RUN_XOR, **T))],
                                         pts=p, out=out, reps=a.reps)
        del out
    if "C3" in only:
        n = 1024
        p = torch.from_numpy(workloads.points(n, workloads.SEED_C3)).cuda()
        out = torch.empty(sm.smap_volume(3, n), dtype=torch.int32, device="cuda")
        var = [("thread_rho8", dict(rho=8, granularity="thread")), ("tile_rho16", dict(rho=16, granularity="tile")),
               ("tile_rho32", dict(rho=32, granularity="tile"))]
        table["configs"]["C3_index_write"] = compare(3, n, "index_write", var + [
            ("tile_rho16_tiles", dict(rho=16, granularity="tile", layout="tiles")),
            ("tile_rho32_tiles", dict(rho=32, granularity="tile", layout="tiles")),
            ("tile_rho32_tiles_xor", dict(rho=32, granularity="tile", layout="tiles", flags=sm.RUN_XOR))],
            out=out, reps=a.reps)
        table["configs"]["C3_atm"] = compare(3, n, "atm", var, pts=p, param=1e-2, reps=a.reps)
        # the config as stated: index write plus ATM sum, fused in one pass
        table["configs"]["C3_index_write_atm"] = compare(3, n, "index_write_atm", var + [
            ("tile_rho16_tiles_xor", dict(rho=16, granularity="tile", layout="tiles", flags=sm.RUN_XOR)),
            ("tile_rho32_tiles_xor", dict(rho=32, granularity="tile", layout="tiles", flags=sm.RUN_XOR))],
            pts=p, param=1e-2, out=out, reps=a.reps)
        del out
    if "C4" in only:
        n = 1 << 17
        out = torch.empty(sm.smap_volume(2, n), dtype=torch.int64, device="cuda")
        table["configs"]["C4"] = compare(2, n, "index_write", [thread2, thread2b, ("tile_rho128", dict(rho=128, granularity="tile")),
                                                                ("tile_rho256", dict(rho=256, granularity="tile")),
                                                                ("tile_rho512", dict(rho=512, granularity="tile")),
                                                                ("tile_rho128_tiles", dict(rho=128, granularity="tile", layout="tiles")),
                                                                ("tile_rho256_tiles", dict(rho=256, granularity="tile", layout="tiles"))],
                                         out=out, reps=max(3, a.reps // 2))
        del out
    if "C5" in only:
        n = 2048
        p = torch.from_numpy(workloads.points(n, workloads.SEED_C5)).cuda()
        var = [("thread_rho8", dict(rho=8, granularity="thread")), ("tile_rho16", dict(rho=16, granularity="tile")),
               ("tile_rho32", dict(rho=32, granularity="tile")), ("tile_rho64", dict(rho=64, granularity="tile")),
               ("tile_rho64_p16", dict(rho=64, granularity="tile", persistent=16)),
               ("tile_rho64_p32", dict(rho=64, granularity="tile", persistent=32))]
        table["configs"]["C5"] = compare(3, n, "tc", var, pts=p, param=0.5, reps=a.reps)
    torch.cuda.empty_cache()
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/configs.json", "w") as f:
        json.dump(table, f, indent=1)


if __name__ == "__main__":
    main()
