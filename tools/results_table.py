#!/usr/bin/env python3
"""Print the DESIGN.md §12 / README results rows from profiles/r02_*.jsonl
(one bench line per workload): info Gbit/s, G edge-updates/s of the decode
kernel, the SFU-model and issue-model fractions."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def lines(path):
    out = []
    for l in open(path):
        l = l.strip()
        if l.startswith("{"):
            out.append(json.loads(l))
    return out


def fracs(d):
    r = d["roofline"]
    sfu = r.get("sfu_model", r)
    issue = r if r["bound"] == "issue" else r.get("issue_model", {})
    return sfu.get("frac"), issue.get("frac"), sfu.get("achieved")


path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02_all_configs.jsonl")
for d in lines(path):
    c = d["config"]
    s, i, a = fracs(d)
    name = c["workload"].split(":")[0]
    print(f"{name:9s} {c['frames_per_step']:>7} frames  {d['value']:7.3f} Gbit/s  {a:7.1f} Gedge-upd/s  "
          f"SFU {s:.3f}  issue {i if i is None else round(i, 3)}  variant {d['roofline'].get('kernel', '')[:40]}")
