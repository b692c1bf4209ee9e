#!/usr/bin/env python3
"""Summarise an `ncu --page source --print-source sass --csv` dump: executed
instructions by opcode, and the hottest basic blocks (runs of instructions
with equal execution counts)."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iex, ismp = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ins = []
for r in rows[2:]:
    try:
        ins.append((r[ia], r[isrc].strip(), int(r[iex]), int(r[ismp])))
    except (ValueError, IndexError):
        pass
tot = sum(x[2] for x in ins)
ops = Counter()
for a, s, n, _ in ins:
    op = s.split()[0] if s else "?"
    if op.startswith("@"):
        op = s.split()[1]
    ops[op.split(".")[0]] += n
print(f"total warp instructions {tot}")
for op, n in ops.most_common(25):
    print(f"  {op:10s} {n:12d} {100*n/tot:5.1f}%")
# blocks
blocks = []
cur = []
for x in ins:
    if cur and x[2] != cur[-1][2]:
        blocks.append(cur); cur = []
    cur.append(x)
if cur:
    blocks.append(cur)
blocks.sort(key=lambda b: -sum(x[2] for x in b))
nshow = int(sys.argv[2]) if len(sys.argv) > 2 else 4
for b in blocks[:nshow]:
    w = sum(x[2] for x in b)
    print(f"\n=== block @{b[0][0]} len {len(b)} exec {b[0][2]} ({100*w/tot:.1f}% of instr), samples {sum(x[3] for x in b)}")
    for a, s, n, smp in b:
        print(f"   {smp:6d}  {s}")
