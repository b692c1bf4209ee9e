#!/usr/bin/env python3
"""Per-source-line instruction and stall totals of one kernel in an ncu report.

    python tools/ncu_lines.py report.ncu-rep <kernel-regex> [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
if rep.endswith(".csv"):      # a source page already exported on the GPU box
    out = open(rep).read()
else:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                          "--kernel-name", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, data = "", None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] and len(r) >= len(hdr) - 1:
        d = dict(zip(hdr[4:], r[4:]))
        d["line"], d["src"], d["file"] = r[0], r[1], fname
        data.append(d)


def num(x):
    try:
        return float(x)
    except (TypeError, ValueError):
        return 0.0


ki, ks = "Instructions Executed", "Warp Stall Sampling (All Samples)"
tot_i = sum(num(d.get(ki)) for d in data)
tot_s = sum(num(d.get(ks)) for d in data)
print(f"total warp instructions {tot_i:.3e}, stall samples {tot_s:.0f}")
for d in sorted(data, key=lambda x: -num(x.get(ki)))[:top]:
    print(f"{d['file']}:{d['line']:>5s} inst {num(d.get(ki))/max(tot_i,1):6.1%} stall {num(d.get(ks))/max(tot_s,1):6.1%}  {d['src'].strip()[:80]}")

# optional: aggregate by line ranges, e.g. RANGES="xf:280-470,crt:690-800,out:840-1010"
import os
rng = os.environ.get("RANGES")
if rng:
    agg = {}
    for part in rng.split(","):
        name, span = part.split(":")
        a, b = (int(v) for v in span.split("-"))
        for d in data:
            if d["file"] == "tc_kernels.cuh" and a <= int(d["line"]) <= b:
                agg.setdefault(name, [0.0, 0.0])
                agg[name][0] += num(d.get(ki)); agg[name][1] += num(d.get(ks))
    other_i = tot_i - sum(v[0] for v in agg.values())
    for k, (i, s) in agg.items():
        print(f"range {k:8s} inst {i/tot_i:6.1%} stall {s/max(tot_s,1):6.1%}")
    fld = [d for d in data if d["file"] == "tc_field.cuh"]
    print(f"tc_field.cuh   inst {sum(num(d.get(ki)) for d in fld)/tot_i:6.1%}")
