#!/usr/bin/env python3
"""profiles/r1_traffic.json and profiles/r1_ncu_metrics.json (read by bench.py for
roofline.traffic / roofline.ncu) from tools/ncu_summary.py text of one
`ncu --set full` capture per config.

    python tools/make_traffic.py C2=profiles/r1_ncu_full_C2_wide.txt C3=profiles/r1_ncu_full_C3.txt
"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1.0, "ms": 1e3, "ns": 1e-3, "s": 1e6}


def stage_of(kernel):
    if "k_low" in kernel:
        return "convert"
    if "k_final" in kernel:
        return "recover"
    m = re.search(r"k_high(?:_ct|_tma)?<(\d)", kernel)
    if m:
        return {"0": "ntt_forward", "1": "ntt_inverse", "2": "pointwise"}[m.group(1)]
    return None


def parse(path):
    out, cur = [], None
    for line in open(path):
        if line.startswith("== "):
            cur = {"kernel": line[3:].split("(")[0].strip()}
            out.append(cur)
            continue
        if cur is None or not line.startswith("   "):
            if not line.strip():
                cur = None
            continue
        parts = line.split()
        if len(parts) >= 2:
            try:
                v = float(parts[1])
            except ValueError:
                continue
            unit = parts[2] if len(parts) > 2 else ""
            cur[parts[0]] = v * UNIT.get(unit, 1.0)
    return out


def main():
    traffic, metrics = {}, {}
    for arg in sys.argv[1:]:
        cfg, path = arg.split("=", 1)
        rel = os.path.relpath(path, ROOT)
        ks = parse(path)
        st, kn = {}, {}
        for k in ks:
            s = stage_of(k["kernel"])
            if s is None or "time" not in k:
                continue
            db = k.get("dram_read", 0.0) + k.get("dram_write", 0.0)
            st.setdefault(s, []).append({"kernel": k["kernel"], "dram_bytes": db, "time_us": round(k["time"], 3)})
            if s not in kn:
                kn[s] = {"kernel": k["kernel"], "time_us": round(k["time"], 3),
                         "issue_active_pct": round(k.get("issue_active_%", 0.0), 1),
                         "pipe_alu_pct": round(k.get("pipe_alu_%", 0.0), 1),
                         "pipe_fma_pct": round(k.get("pipe_fma_%", 0.0), 1),
                         "occupancy_pct": round(k.get("occupancy_%", 0.0), 1),
                         "dram_gbs": round(db / (k["time"] * 1e-6) / 1e9, 1)}
        src = f"{rel} (ncu --set full --clock-control none, one capture)"
        traffic[cfg] = {"source": src, "stages": st}
        metrics[cfg] = {"source": rel, "kernels": kn}
    json.dump(traffic, open(os.path.join(ROOT, "profiles", os.environ.get("TAG", "r2") + "_traffic.json"), "w"), indent=1)
    json.dump(metrics, open(os.path.join(ROOT, "profiles", os.environ.get("TAG", "r2") + "_ncu_metrics.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
