#!/usr/bin/env python3
"""Summarise an `ncu --page source --csv --print-source sass` dump: executed
instructions by opcode, and the instructions with the most stall samples
(per stall reason).   python tools/sass_hot.py dump.csv [top]"""
import csv
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


ops = Counter()
samples = Counter()
stalls = defaultdict(Counter)
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot_inst = 0.0
tot_samp = 0.0
for r in data:
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    n = num(r[ix["Instructions Executed"]])
    ops[op] += n
    tot_inst += n
    s = num(r[ix["Warp Stall Sampling (All Samples)"]])
    tot_samp += s
    samples[(r[ix["Address"]], src)] += s
    for rs in reasons:
        stalls[rs][op] += num(r[ix[rs]])
print(f"# {len(data)} SASS lines, {tot_inst:.4g} warp instructions, {tot_samp:.4g} stall samples")
print("## executed warp instructions by opcode")
for op, n in ops.most_common(top):
    print(f"{op:12s} {n:14.4g} {100 * n / tot_inst:6.2f}%")
print("## stall samples by reason (and the opcodes they sit on)")
tot_r = {rs: sum(c.values()) for rs, c in stalls.items()}
for rs, t in sorted(tot_r.items(), key=lambda x: -x[1])[:10]:
    if t <= 0:
        continue
    tops = ", ".join(f"{o} {100 * v / t:.0f}%" for o, v in stalls[rs].most_common(4))
    print(f"{rs:22s} {100 * t / tot_samp:6.2f}%   [{tops}]")
print("## hottest instructions (stall samples)")
for (addr, src), s in samples.most_common(top):
    print(f"{100 * s / tot_samp:6.2f}%  {src[:90]}")
