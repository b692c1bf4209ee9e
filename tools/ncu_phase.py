#!/usr/bin/env python3
"""Instruction / stall-sample totals of a kernel's source page grouped by source line ranges.
    python tools/ncu_phase.py fin_src.csv"""
import csv, sys, collections
rows = csv.reader(open(sys.argv[1]))
fname = ""; hdr = None; seen = set(); inst = collections.Counter(); stall = collections.Counter()
per_line = {}
def _ranges():
    """Line ranges of the kernels' phases, from the current source."""
    import os, re
    src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1612_05778_b200", "csrc",
                            "tc_kernels.cuh")).read().split("\n")
    def at(pat, start=0):
        for i in range(start, len(src)):
            if re.search(pat, src[i]): return i + 1
        return len(src)
    marks = [("digits", r"struct DigitSrc"), ("other0", r"static __global__ void __launch_bounds__\(256\) k_digits"),
             ("generic-round", r"struct LanePerm"), ("x-round", r"void xct_round"), ("y-round", r"void yct_round"),
             ("y-expand", r"void yct_expand_columns"), ("other1", r"struct TwRows"), ("k_low-body", r"struct LowArgs"),
             ("k_high", r"enum \{ MODE_FWD"), ("crt", r"struct CrtConst"), ("other2", r"int div_m\("),
             ("co-grouped", r"struct WordAcc"), ("co-pieces", r"void warp_term_pieces"), ("co-warp", r"void crt_convert_warp"),
             ("co-words", r"void convert_out_words"), ("k_final-body", r"FinalArgs A, const __grid_constant__ CrtConst"),
             ("other3", r"void k_unshard")]
    pos = [(at(pat), name) for name, pat in marks]
    out = []
    for i, (ln, name) in enumerate(pos):
        end = pos[i + 1][0] - 1 if i + 1 < len(pos) else len(src)
        out.append((ln, end, name))
    return out
RANGES = _ranges()
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
        if 44 <= l <= 70: return "bfly-alu"
        if l in (39, 40): return "shoup_mul"
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
