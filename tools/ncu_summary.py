#!/usr/bin/env python
"""Summarise ncu output for profiles/ (run here, on the CPU box).

usage: ncu_summary.py launches <launches.csv> [k1,k2]  per-kernel launch times + step share
                                                       (over the kernels named, default every
                                                       k_scan / k_slide / k_estimate*)
       ncu_summary.py full <report.ncu-rep> [label]    key metrics per profiled kernel
       ncu_summary.py traffic <report.ncu-rep> <key>   dram bytes per launch (json fragment)
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors.sum",
    "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
    "lts__t_requests_op_red.sum", "lts__t_sectors_op_red.sum", "lts__t_requests_op_atom.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
]


def short(name: str) -> str:
    base = name.split("(")[0]
    return base.replace("void ", "").replace("<unnamed>::", "")


def launches(path, only=None):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[h + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        k = short(r[ki])
        tot[k] += float(r[vi].replace(",", ""))
        cnt[k] += 1
    pick = tuple(only.split(",")) if only else ("k_scan", "k_slide", "k_estimate")
    step = {k: tot[k] / cnt[k] for k in tot if k.startswith(pick)}
    s = sum(step.values())
    print(f"{'avg ns':>12} {'count':>6} {'share of step':>14}  kernel")
    for k in sorted(tot, key=lambda k: -tot[k] / cnt[k]):
        share = f"{100 * step[k] / s:.1f}%" if k in step else "-"
        print(f"{tot[k] / cnt[k]:12.0f} {cnt[k]:6d} {share:>14}  {k}")


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def full(rep, label=""):
    hdr, units, rows = raw(rep)
    ki = hdr.index("Kernel Name")
    print(f"# ncu --set full summary {label} ({rep})")
    for r in rows:
        print(f"\n## {short(r[ki])}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:75s} {r[i]:>16s} {units[i]}")


def traffic(rep, key_prefix):
    hdr, units, rows = raw(rep)
    ki = hdr.index("Kernel Name")
    rd, wr = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    out = {}
    for r in rows:
        name = short(r[ki])
        kind = ("scan" if name.startswith("k_scan") else "slide" if name.startswith("k_slide")
                else "estimate_plan" if name.startswith("k_estimate_plan")
                else "estimate" if name.startswith("k_estimate") else None)
        if kind:
            b = float(r[rd]) * scale[units[rd]] + float(r[wr]) * scale[units[wr]]
            out[f"{key_prefix}/{kind}"] = int(b)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "launches":
        launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
    elif cmd == "full":
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
    elif cmd == "traffic":
        traffic(sys.argv[2], sys.argv[3])
