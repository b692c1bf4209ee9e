#!/usr/bin/env python3
"""Instruction / stall-sample totals of a kernel's source page grouped by source line ranges.
    python tools/ncu_phase.py fin_src.csv"""
import csv, sys, collections
rows = csv.reader(open(sys.argv[1]))
fname = ""; hdr = None; seen = set(); inst = collections.Counter(); stall = collections.Counter()
per_line = {}
RANGES = [(225, 470, "digits"), (640, 745, "x-round"), (746, 925, "y-round"), (926, 1000, "y-expand"), (1064, 1128, "k_low-body"), (1129, 1146, "k_low-residues"), (1147, 1218, "k_low-body"),
          (1757, 1812, "crt"), (2126, 2178, "co-pieces"), (2179, 2335, "co-warp"), (2472, 2650, "k_final-body")]
stall_kinds = collections.defaultdict(collections.Counter)
for r in rows:
    if not r: continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name": continue
    if r[0] == "Line No": hdr = r; continue
    if not hdr or not r[0] or not r[0].isdigit(): continue
    key = (fname, int(r[0]))
    if key in seen: continue       # second kernel instance
    seen.add(key)
    d = dict(zip(hdr[4:], r[4:]))
    try:
        ni = float(d["Instructions Executed"]); ns = float(d["# Samples"])
    except ValueError: continue
    per_line[key] = (ni, ns, r[1], d)
def cat(f, l):
    if f == "tc_field.cuh":
        if 60 <= l <= 75: return "bfly-alu"
        if l in (33, 34): return "shoup_mul"
        return "field-other"
    if f == "tc_kernels.cuh":
        for lo, hi, name in RANGES:
            if lo <= l <= hi: return name
        return "kern-other"
    return f
ti = sum(v[0] for v in per_line.values()); ts = sum(v[1] for v in per_line.values())
for k, (ni, ns, src, d) in per_line.items():
    c = cat(*k); inst[c] += ni; stall[c] += ns
    for name in ("stall_barrier","stall_long_sb","stall_math","stall_mio","stall_not_selected","stall_selected","stall_short_sb","stall_wait","stall_lg","stall_dispatch","stall_branch_resolving","stall_no_inst"):
        try: stall_kinds[c][name] += float(d[name])
        except (KeyError, ValueError): pass
print(f"total warp inst {ti:.3e} samples {ts:.0f}")
for c in sorted(inst, key=lambda c: -inst[c]):
    top = ", ".join(f"{k[6:]} {v/ max(stall[c],1)*100:.0f}%" for k, v in stall_kinds[c].most_common(5))
    print(f"{c:16s} inst {inst[c]/ti*100:5.1f}%  samples {stall[c]/ts*100:5.1f}%   [{top}]")
