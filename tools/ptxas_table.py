#!/usr/bin/env python3
"""Per-kernel registers / spills from `nvcc -Xptxas -v` logs (build/*.ptxas.log):
    python tools/ptxas_table.py LOG [OLD_LOG]   (with OLD_LOG: only kernels that changed)"""
import re
import subprocess
import sys


def parse(path):
    out, cur = {}, None
    for line in open(path):
        m = re.search(r"Compiling entry function '([^']+)'", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur:
            out.setdefault(cur, {})["spill"] = (int(m.group(1)), int(m.group(2)))
        m = re.search(r"Used (\d+) registers", line)
        if m and cur:
            out.setdefault(cur, {})["regs"] = int(m.group(1))
    return out


def demangle(names):
    try:
        p = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
        return p.stdout.splitlines()
    except Exception:
        return names


new = parse(sys.argv[1])
old = parse(sys.argv[2]) if len(sys.argv) > 2 else None
names = sorted(new)
dm = dict(zip(names, demangle(names)))
for k in names:
    v = new[k]
    o = old.get(k) if old else None
    if old is not None and o == v:
        continue
    d = dm[k].replace("(anonymous namespace)::", "")
    d = re.sub(r"\(.*$", "", d)[:90]
    tail = f"   (was {o.get('regs')} regs, spill {o.get('spill')})" if o else ""
    print(f"{v.get('regs', '?'):>4} regs spill {str(v.get('spill')):>12}  {d}{tail}")
