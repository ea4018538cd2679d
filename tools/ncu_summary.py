#!/usr/bin/env python
"""Summarise ncu outputs into profiles/: a launch list (gpu__time_duration per
launch, share of the step) and the key counters of a --set full capture.

  python tools/ncu_summary.py --launches gpurun_out/launches_c2.csv \
      --report gpurun_out/prof_c2.ncu-rep --name C2 --grid 512 512 512 --round r01
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum.per_second",
    "dram__bytes_write.sum.per_second", "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "lts__t_bytes.sum",
    "smsp__average_warp_latency_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "s": 1, "usecond": 1e-6, "nsecond": 1e-9, "msecond": 1e-3}


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1)
                out.append((d["Kernel Name"], v))
    return out


def raw(report):
    """Counters of a --set full capture: an .ncu-rep (exported here) or its raw-page CSV export."""
    if report.endswith(".csv"):
        txt = open(report).read()
    else:
        txt = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        e = {"kernel": d.get("Kernel Name", "")}
        for k in KEYS:
            if k in d and d[k] != "":
                u = units[hdr.index(k)]
                try:
                    val = float(d[k].replace(",", ""))
                except ValueError:
                    continue
                e[k] = {"value": val, "unit": u}
        res.append(e)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--report")
    ap.add_argument("--name", required=True)
    ap.add_argument("--grid", type=int, nargs=3, required=True)
    ap.add_argument("--round", default="r01")
    ap.add_argument("--bytes-per-point", type=float, default=36.0)
    ap.add_argument("--key", default=None, help="entry name in profiles/ncu_summary.json (default --name)")
    a = ap.parse_args()
    out = {"config": a.name, "grid": a.grid, "round": a.round}
    npts = a.grid[0] * a.grid[1] * a.grid[2]
    if a.launches:
        L = launches(a.launches)
        agg = defaultdict(list)
        for k, v in L:
            agg[k].append(v)
        tot = sum(v for _, v in L)
        out["launch_list"] = {k: {"launches": len(v), "mean_s": sum(v) / len(v), "share_of_listed_time": sum(v) / tot}
                              for k, v in agg.items()}
    if a.report:
        R = raw(a.report)
        out["full_set"] = R
        step = [e for e in R if "vti_step_kernel" in e["kernel"]]
        if step:
            rd = sum(e["dram__bytes_read.sum"]["value"] * SCALE[e["dram__bytes_read.sum"]["unit"]] for e in step) / len(step)
            wr = sum(e["dram__bytes_write.sum"]["value"] * SCALE[e["dram__bytes_write.sum"]["unit"]] for e in step) / len(step)
            t = sum(e["gpu__time_duration.sum"]["value"] * SCALE[e["gpu__time_duration.sum"]["unit"]] for e in step) / len(step)
            out["step_kernel"] = {
                "dram_read_bytes": rd, "dram_write_bytes": wr, "dram_bytes_per_launch": rd + wr,
                "algorithmic_bytes_per_launch": a.bytes_per_point * npts,
                "traffic_over_algorithmic": (rd + wr) / (a.bytes_per_point * npts),
                "dram_bytes_per_point": (rd + wr) / npts, "duration_s": t, "dram_GBps": (rd + wr) / t / 1e9,
            }
    key = a.key or a.name
    path = os.path.join("profiles", f"ncu_{key}_{a.round}.json")
    json.dump(out, open(path, "w"), indent=1)
    summ = os.path.join("profiles", "ncu_summary.json")
    s = json.load(open(summ)) if os.path.exists(summ) else {}
    if "step_kernel" in out:
        s[key] = {"grid": a.grid, "round": a.round, "dram_bytes_per_launch": out["step_kernel"]["dram_bytes_per_launch"],
                     "source": os.path.basename(path)}
        json.dump(s, open(summ, "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "full_set"}, indent=1))


if __name__ == "__main__":
    main()
