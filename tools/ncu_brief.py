#!/usr/bin/env python3
"""One line per kernel of an .ncu-rep: time, issue, occupancy, conflicts, stalls."""
import csv
import subprocess
import sys

WANT = {
    "time_us": "gpu__time_duration.sum",
    "issue%": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps%": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "blk/SM": "launch__occupancy_limit_shared_mem",
    "bankconf": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "shm_wavefr": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "inst": "smsp__inst_executed.sum",
    "dramMB_r": "dram__bytes_read.sum",
    "dramMB_w": "dram__bytes_write.sum",
}
STALLS = ["long_scoreboard", "short_scoreboard", "wait", "mio_throttle", "barrier", "math_pipe_throttle",
          "lg_throttle", "not_selected", "selected", "dispatch_stall", "no_instruction", "branch_resolving"]

for path in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")][:34]
        vals = []
        for k, m in WANT.items():
            v = r[hdr.index(m)] if m in hdr else "?"
            vals.append(f"{k}={v}")
        st = []
        for s in STALLS:
            m = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if m in hdr:
                try:
                    st.append(f"{s}={float(r[hdr.index(m)]):.2f}")
                except ValueError:
                    pass
        print(name, " ".join(vals))
        print("    stalls/issue:", " ".join(st))
