#!/usr/bin/env python3
"""Print a one-line-per-config table from bench.py JSON lines."""
import json
import sys

for line in open(sys.argv[1]):
    line = line.strip()
    if not line.startswith("{"):
        if line and ("Error" in line or "error" in line):
            print("   ", line[:300])
        continue
    d = json.loads(line)
    c = d["config"]
    e2e = d.get("e2e") or {}
    print(f"{c['workload'][:8]:8s} n={c['n']:<6d} F={c['frames_per_gpu_per_step']:<7d} {d['value']:7.3f} Gb/s "
          f"dec={d['decode_ms_per_step']:9.2f} ms frac={d['roofline']['frac']:.3f} "
          f"ach={d['roofline']['achieved']:6.1f} it={d['mean_iterations']:5.2f} "
          f"e2e={e2e.get('value') or 0:.3f} step={d['ms_per_step']:.2f} clk={d['clocks']['sm_mhz']}")
