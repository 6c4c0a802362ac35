#!/usr/bin/env python3
"""Summarise an ncu report (--set full) or a launch-list CSV for profiles/.

    python scripts/ncu_summary.py report gpurun_out/prof_full.ncu-rep [--json out.json]
    python scripts/ncu_summary.py launches gpurun_out/ncu_launches.csv
"""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict

DETAILS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate",
           "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "Compute (SM) Throughput",
           "Issue Slots Busy", "Grid Size", "Block Size", "Waves Per SM", "Dynamic Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct", "gpu__time_duration.sum",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def ncu_csv(args):
    out = subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def report(path):
    res = OrderedDict()
    rows = ncu_csv(["-i", path, "--page", "details", "--csv"])
    h = rows[0]
    ki, idi, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
    for r in rows[1:]:
        key = f"{r[idi]}:{r[ki].split('(')[0].replace('<unnamed>::', '').replace('void ', '')}"
        if r[mi] in DETAILS:
            res.setdefault(key, OrderedDict())[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    raw = ncu_csv(["-i", path, "--page", "raw", "--csv"])
    h = raw[0]
    for r in raw[2:]:
        if len(r) != len(h):
            continue
        key = f"{r[h.index('ID')]}:{r[h.index('Kernel Name')].split('(')[0].replace('<unnamed>::', '').replace('void ', '')}"
        d = res.setdefault(key, OrderedDict())
        for m in RAW:
            if m in h:
                d[m] = r[h.index(m)]
        stalls = []
        for i, name in enumerate(h):
            if name.startswith("smsp__average_warp_latency_issue_stalled_") or \
               (name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("_not_issued")):
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                if v > 0:
                    stalls.append((v, name.split("stalled_")[-1]))
        stalls.sort(reverse=True)
        d["top_stalls(pc samples)"] = ", ".join(f"{n}={int(v)}" for v, n in stalls[:6])
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    idx = {x: j for j, x in enumerate(h)}
    data = OrderedDict()
    for r in rows[start + 1:]:
        if len(r) < len(h):
            continue
        key = (int(r[idx["ID"]]), r[idx["Kernel Name"]].split("(")[0].replace("<unnamed>::", "").replace("void ", ""))
        data.setdefault(key, {})[r[idx["Metric Name"]]] = float(r[idx["Metric Value"]].replace(",", ""))
    return data


def main():
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "report":
        res = report(path)
        for k, d in res.items():
            print(f"== {k}")
            for m, v in d.items():
                print(f"   {m}: {v}")
        if "--json" in sys.argv:
            json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
    else:
        data = launches(path)
        tot = sum(d.get("gpu__time_duration.sum", 0) for d in data.values())
        print(f"{'id':>4} {'kernel':42} {'time_us':>10} {'share':>7} {'dram_rd_MB':>11} {'dram_wr_MB':>11} {'GB/s':>8}")
        for (i, name), d in data.items():
            t = d.get("gpu__time_duration.sum", 0)
            rd, wr = d.get("dram__bytes_read.sum", 0), d.get("dram__bytes_write.sum", 0)
            print(f"{i:>4} {name[:42]:42} {t / 1e3:>10.1f} {t / tot:>7.1%} {rd / 1e6:>11.1f} {wr / 1e6:>11.1f} "
                  f"{(rd + wr) / max(t, 1):>8.0f}")


if __name__ == "__main__":
    main()
