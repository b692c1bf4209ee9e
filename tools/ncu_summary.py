#!/usr/bin/env python3
"""Summarise an ncu report (.ncu-rep) or a launch-list CSV for profiles/.

    python tools/ncu_summary.py report.ncu-rep      # key metrics per profiled launch
    python tools/ncu_summary.py launches.csv        # per-kernel time share
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_throughput_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_%"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "pipe_alu_%"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "pipe_fma_%"),
    ("sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active", "pipe_fmaheavy_%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "pipe_lsu_%"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu_cycles_%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_cycles_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
    ("smsp__inst_executed.sum", "warp_insts"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    for r in data:
        print(f"== {r[idx['Kernel Name']][:90]}")
        for key, label in KEYS:
            if key in idx:
                print(f"   {label:22s} {r[idx[key]]} {units[idx[key]]}")
        stalls = [(h, r[i]) for h, i in idx.items()
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
        vals = []
        for h, v in stalls:
            try:
                vals.append((float(v.replace(",", "")), h))
            except ValueError:
                pass
        tot = sum(v for v, _ in vals) or 1.0
        for v, h in sorted(vals, reverse=True)[:8]:
            print(f"   stall {h.split('stalled_')[-1]:28s} {v / tot:6.1%}")


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[mi], 1.0)
        name = r[ki].split("(")[0]
        tot[name] += v * scale
        cnt[name] += 1
    s = sum(tot.values())
    print(f"{'kernel':40s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}")
    for k in sorted(tot, key=tot.get, reverse=True):
        print(f"{k[:40]:40s} {cnt[k]:8d} {tot[k]:10.1f} {tot[k]/cnt[k]:9.2f} {tot[k]/s:6.1%}")


if __name__ == "__main__":
    p = sys.argv[1]
    (report if p.endswith(".ncu-rep") else launches)(p)
