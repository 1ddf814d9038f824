"""Summarise an ncu --set full capture into the JSON kept under profiles/.

    python scripts/ncu_summary.py gpurun_out/x.ncu-rep profiles/r01_x_ncu_full.json [--traffic-key '<cfg json>']

Reads `ncu -i <rep> --page raw --csv` (one row per captured kernel; the last
one is summarised) and keeps the metrics DESIGN.md and bench.py cite: time,
DRAM bytes and throughput, issue activity, pipe utilisation, occupancy, the
top stall reasons.  With --traffic-key the DRAM read+write bytes are also
recorded in profiles/ncu_traffic.json under that key (bench.py's `traffic`).
"""
import argparse
import csv
import io
import json
import os
import subprocess

KEEP = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second", "lts__t_sectors_srcunit_tex_op_write.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--traffic-key", default=None)
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[-1]
    col = {h: i for i, h in enumerate(hdr)}
    summ = {"Kernel Name": vals[col["Kernel Name"]]}
    for k in KEEP:
        if k in col:
            summ[k] = f"{vals[col[k]]} {units[col[k]]}".strip()
    stalls = {}
    for h, i in col.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(vals[i])
            except ValueError:
                pass
    summ["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
    try:
        rd = float(vals[col["dram__bytes_read.sum"]]) * UNIT_SCALE.get(units[col["dram__bytes_read.sum"]], 1)
        wr = float(vals[col["dram__bytes_write.sum"]]) * UNIT_SCALE.get(units[col["dram__bytes_write.sum"]], 1)
        summ["traffic_bytes_per_launch"] = rd + wr
    except (KeyError, ValueError):
        rd = wr = None
    with open(a.out, "w") as f:
        json.dump(summ, f, indent=1)
    if a.traffic_key and rd is not None:
        path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
        tr = json.load(open(path)) if os.path.exists(path) else {}
        tr[a.traffic_key] = rd + wr
        with open(path, "w") as f:
            json.dump(tr, f, indent=1)
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main()
