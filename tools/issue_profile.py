#!/usr/bin/env python3
"""Issue-slot profile of the decode kernel per workload (issue
budget <= 32 thread-instructions per edge-update at 100% of the SFU price).

For each workload, one ncu pass over ONE decode launch of the bench's own
launch configuration (bench.py --eager: the first decode launch of the step):
    smsp__inst_executed.sum          warp instructions issued
    smsp__thread_inst_executed.sum   thread instructions (active lanes)
    sm__inst_executed_pipe_xu.sum    MUFU (XU pipe) warp instructions
    smsp__issue_active.avg.pct_of_peak_sustained_active
    launch__grid_size, gpu__time_duration.sum
The same run's bench JSON line gives the launch's edge-updates (frames x
edges x mean iterations).  Writes profiles/issue.json (read by bench.py's
roofline) and prints a table.  Run on the GPU box:
    python tools/issue_profile.py [out.json]
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import ldpc_workloads as W  # noqa: E402

METRICS = ["smsp__inst_executed.sum", "smsp__thread_inst_executed.sum", "sm__inst_executed_pipe_xu.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "gpu__time_duration.sum"]
# (workload, frames of the bench launch, extra bench args): the bench's own
# launch per config (bench_all.sh sizes; C5 = one 16,384-frame chunk)
RUNS = [("C1", 1000, []), ("C2", 10000, ["--ebn0", "1.0"]), ("C3-R1/4", 100000, []), ("C3-R1/2", 100000, []),
        ("C3-R3/4", 100000, []), ("C4", 200000, []), ("C5", 16384, []), ("T1-R1/4", 1000, []),
        ("T1-R1/2", 1000, []), ("T1-R3/4", 1000, [])]
KREGEX = "regex:band_kernel|xband|edge_kernel|spa_decode_kernel|band_cluster"


def run(cfg, frames, extra):
    cmd = ["ncu", "--csv", "--clock-control", "none", "--metrics", ",".join(METRICS), "-k", KREGEX, "-c", "1",
           sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--frames", str(frames), "--steps", "1",
           "--warmup", "0", "--eager", "--no-cpu-baseline", "--no-e2e", *extra]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=1800)
    out = p.stdout
    line = next((json.loads(l) for l in out.splitlines() if l.startswith('{"metric"')), None)
    rows = [l for l in out.splitlines() if l.startswith('"')]
    vals, kname, hdr = {}, None, None
    for r in csv.reader(io.StringIO("\n".join(rows))):
        if r and r[0] == "ID":
            hdr = {name: i for i, name in enumerate(r)}
            continue
        if not hdr or len(r) < len(hdr):
            continue
        kname = r[hdr["Kernel Name"]]
        try:
            vals[r[hdr["Metric Name"]]] = float(r[hdr["Metric Value"]].replace(",", ""))
        except ValueError:
            pass
    return line, vals, kname, p.returncode, p.stderr[-2000:]


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "issue.json")
    # optional second argument: a comma list of workloads to re-measure, merged
    # into the existing file (the others keep their entries)
    only = set(sys.argv[2].split(",")) if len(sys.argv) > 2 else None
    prev = {}
    if only and os.path.exists(out_path):
        with open(out_path) as f:
            prev = json.load(f)
    res = dict(prev)
    res |= {"_source": "tools/issue_profile.py: ncu --metrics " + ",".join(METRICS) +
                      " over one decode launch of bench.py's launch configuration per workload; "
                      "thread_instructions_per_edge_update = 32 x warp instructions / edge-updates "
                      "(issue slots, full warps); active_lane_instructions_per_edge_update = thread "
                      "instructions (active lanes) / edge-updates"}
    for cfg, frames, extra in RUNS:
        if only and cfg not in only:
            continue
        line, vals, kname, rc, err = run(cfg, frames, extra)
        if not line or "smsp__inst_executed.sum" not in vals:
            print(f"{cfg}: failed rc={rc} {err}", flush=True)
            continue
        wl = W.ALL[cfg]
        ctr = line["counters"]
        eu = ctr["frames"] * wl.edges * line["mean_iterations"]
        wi = vals["smsp__inst_executed.sum"]
        e = {"frames": frames, "kernel": kname, "edge_updates": eu,
             "thread_instructions_per_edge_update": 32.0 * wi / eu,
             "active_lane_instructions_per_edge_update": vals.get("smsp__thread_inst_executed.sum", 0.0) / eu,
             "mufu_per_edge_update": 32.0 * vals.get("sm__inst_executed_pipe_xu.sum", 0.0) / eu,
             "issue_active_pct": vals.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
             "grid": vals.get("launch__grid_size"), "ncu_duration_ns": vals.get("gpu__time_duration.sum"),
             "source": f"profiles/issue.json ({cfg}, {frames} frames, ncu {'/'.join(m.split('.')[0] for m in METRICS[:3])})"}
        if extra:
            e["bench_args"] = " ".join(extra)
        res[cfg] = e
        print(f"{cfg:8s} {frames:7d} frames: {e['thread_instructions_per_edge_update']:6.2f} issue-slot "
              f"thread-instr/edge-update, {e['mufu_per_edge_update']:5.2f} MUFU/edge-update, issue active "
              f"{e['issue_active_pct']}%  [{kname[:60]}]", flush=True)
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
