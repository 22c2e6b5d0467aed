#!/usr/bin/env python3
"""Summarise ncu outputs for profiles/: a launch list (--metrics
gpu__time_duration.sum --csv) and the key counters of a --set full report."""
import csv
import subprocess
import sys
from collections import defaultdict

UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows[hi + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        ms = float(d["Metric Value"].replace(",", "")) * UNIT[d["Metric Unit"]]
        name = d["Kernel Name"].split("(")[0].replace("void ", "")[:70]
        agg[name][0] += 1
        agg[name][1] += ms
        total += ms
    print(f"# ncu launch list: {sum(c for c, _ in agg.values())} launches, {total:.1f} ms total (cold-cache, serialised)")
    print(f"{'launches':>8} {'total ms':>12} {'mean ms':>10} {'share':>7}  kernel")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{c:8d} {t:12.3f} {t / c:10.3f} {100 * t / total:6.1f}%  {k}")


KEYS = ["Duration", "SM Frequency", "Elapsed Cycles", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block",
        "Achieved Occupancy", "Theoretical Occupancy", "Warp Cycles Per Issued Instruction",
        "Eligible Warps Per Scheduler", "Executed Instructions", "L1/TEX Hit Rate", "L2 Hit Rate"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
       "smsp__average_warp_latency_issue_stalled_barrier", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    seen = set()
    name = None
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        name = name or d.get("Kernel Name")
        m = d.get("Metric Name")
        if m in KEYS and m not in seen:
            seen.add(m)
            print(f"{m:40s} {d.get('Metric Value'):>18s} {d.get('Metric Unit')}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    h, units, vals = rr[0], rr[1], rr[2]
    for k in RAW:
        for i, col in enumerate(h):
            if col == k:
                print(f"{k:60s} {vals[i]:>18s} {units[i]}")
    # stall reasons
    for i, col in enumerate(h):
        if col.startswith("smsp__average_warps_issue_stalled_") and col.endswith("_per_issue_active.ratio"):
            try:
                v = float(vals[i].replace(",", ""))
            except ValueError:
                continue
            if v >= 0.2:
                print(f"stall {col[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:28s} {v:8.2f}")
    print(f"# kernel: {name}")


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    launches(path) if mode == "launches" else full(path)
