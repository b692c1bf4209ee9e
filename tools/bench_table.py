#!/usr/bin/env python3
"""Print a compact table of bench JSON lines (gpurun_out/bench_C*.json)."""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as ex:  # noqa: BLE001
        print(path, "unreadable", ex)
        continue
    c = d["config"]
    print(f"{c['workload'][:60]:60s} dev {d['ms_per_step']:9.4f} ms  {d['value']:8.2f} Gbit/s | "
          f"e2e {d['e2e']['ms_per_step']:9.4f} ms {d['e2e']['value']:8.2f} | verified={c.get('verified_vs_reference_sha256')} "
          f"launches={d.get('gpu_launches')}")
    print(f"    plan: {c['plan']}")
    for k, v in d["roofline"]["stages"].items():
        print(f"    {k:12s} {v['ms']:9.4f} ms  {v['GBps']:8.1f} GB/s ({v['hbm_frac']:.3f})  "
              f"{v['Gbfly_s']:8.1f} Gbfly/s ({v['int_frac']})")
