#!/usr/bin/env python3
"""Benchmark: product time and output Gbit/s of the dense Z[y] multiply on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--extra C1,C2,C4,C5]
                    [--impl ours|reference]

Metric (BASELINE.json): "product time (ms) & output Gbit/s, dxN-bit Z[x]
multiply"; `value` is output Gbit/s = rows*out_bits/1e9 per product / time.
Workload: BASELINE config C3 (d=65536, N=65536-bit, half all-ones), the
largest configuration that fits one GPU (BASELINE.json's metric names no
single config); C1, C2, C4, C5 are measured beside it (`other_configs`).
Seeded synthetic inputs (paper_1612_05778_b200/workloads.py), the same arrays
the reference hashes in tests/golden/configs.json; every config's product is
checked against the reference's SHA-256 before it is timed.

* value      device-resident: inputs already in HBM, output left in HBM; each
             step = device width scan + every kernel, timed with CUDA events on
             the library's stream, L2 flushed (256 MiB memset) before every step
             outside the timed region.
* e2e        the public API `multiply(MulRequest(a, b))` on plain (pageable)
             numpy arrays, as a drop-in caller holds them: H2D of both operands,
             all kernels and D2H of the product inside the timed region (wall
             clock around the synchronous call).  `e2e_pinned`: page-locked inputs.
* roofline   every stage of the device-resident step: algorithmic bytes (HBM)
             and radix-2 butterflies (INT pipe) / its event time, against
             MEASURED_PEAKS.json's HBM copy bandwidth and the butterfly peak
             measured live by tc_int_peak; the longest stage is the headline.
* cpu_baseline  the reference's algorithm (oracle/, a C restatement of its numba
             kernels, 63-bit primes, its own plan) on this host: one full product
             on all cores with the stage split, and a one-thread sample.

`--impl reference` times that same CPU restatement as the reference arm.
N > 1 (torchrun): ONE product sharded over the N GPUs (shard.py); "scaling":
"strong", time = max over ranks of CUDA-event time on each rank.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1612_05778_b200 import workloads  # noqa: E402

METRIC = "product time (ms) & output Gbit/s, dxN-bit Z[x] multiply, at 1/2/4/8 B200"


def _dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


class ClockSampler:
    """SM clock + throttle reasons sampled during the measured loops: NVML
    polled every 2 ms from a background thread (nvidia-smi -lms 50 when NVML
    is unavailable)."""

    def __init__(self, device: int):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [x for x in vis.split(",") if x.strip()]
        self.index = int(ids[device]) if device < len(ids) and ids[device].strip().isdigit() else device
        self.samples, self.reason_bits, self.max_mhz = [], 0, None
        self.stop_evt = threading.Event()
        self.proc = None
        self.lines = []
        self.nvml = None

    def start(self, wait_s: float = 5.0):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.nvml = (pynvml, h)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.samples and time.time() - t0 < wait_s:
                time.sleep(0.001)
            return
        except Exception:  # noqa: BLE001 -- fall back to nvidia-smi
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < wait_s:
                time.sleep(0.01)
        except (OSError, FileNotFoundError):
            self.proc = None

    def _poll(self):
        pynvml, h = self.nvml
        get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop_evt.is_set():
            try:
                self.samples.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                self.reason_bits |= int(get_reasons(h))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = set()
        if self.nvml:
            self.stop_evt.set()
            self.thread.join(timeout=2)
            pynvml = self.nvml[0]
            bits = (pynvml.nvmlClocksThrottleReasonHwSlowdown, pynvml.nvmlClocksThrottleReasonHwThermalSlowdown,
                    pynvml.nvmlClocksThrottleReasonSwThermalSlowdown, pynvml.nvmlClocksThrottleReasonSwPowerCap)
            for n, b in zip(names, bits):
                if self.reason_bits & b:
                    reasons.add(n)
            sm, mx, src = self.samples, self.max_mhz, "nvml, 2 ms"
        else:
            if self.proc:
                self.proc.terminate()
                try:
                    self.proc.wait(timeout=5)
                except subprocess.TimeoutExpired:
                    self.proc.kill()
            sm, mx, src = [], None, "nvidia-smi, 50 ms"
            for ln in self.lines:
                parts = [x.strip() for x in ln.split(",")]
                if len(parts) < 6:
                    continue
                try:
                    sm.append(float(parts[0]))
                    mx = float(parts[1])
                except ValueError:
                    continue
                for n, v in zip(names, parts[2:6]):
                    if v.lower() == "active":
                        reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(sm)), "sm_min_mhz": float(np.min(sm)), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "sampler": src}


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


def stage_model(plan, da, db, a_cw, b_cw, out_cw):
    """Algorithmic HBM bytes and radix-2 butterflies of each pipeline stage,
    for the pass layout the library runs (params.pass_layout == make_geometry
    in csrc/tc_api.cu).  Butterflies are the canonical count (zero padding
    not pruned); bytes are one read of each input and one write of each output
    of every kernel in the stage."""
    from paper_1612_05778_b200.params import pass_layout
    P, L, s_y = plan.P, plan.L, plan.s_y
    S = s_y * L
    lgL = L.bit_length() - 1
    lgS = s_y.bit_length() - 1
    rows = da + db - 1
    yl, high = pass_layout(lgL, lgS, P)
    low_bits = lgL + yl
    g = 4 * P * S                      # one sweep over one operand's P grids
    st = {}
    st["convert"] = dict(bytes=(da * a_cw + db * b_cw) * 8 + 2 * g, bfly=2 * P * (S // 2) * low_bits)
    fb = ff = 0
    for i, (u0, U) in enumerate(high):
        for op in ("A", "B"):
            if op == "B" and i == len(high) - 1:
                continue
            fb += 2 * g
            ff += P * (S // 2) * U
    st["ntt_forward"] = dict(bytes=fb, bfly=ff)
    u_last = high[-1][1] if high else 0
    st["pointwise"] = dict(bytes=3 * g, bfly=2 * P * (S // 2) * u_last)
    st["ntt_inverse"] = dict(bytes=2 * g * max(len(high) - 1, 0),
                             bfly=sum(P * (S // 2) * U for (_, U) in high[:-1]))
    st["recover"] = dict(bytes=g + 8 * rows * out_cw, bfly=P * (S // 2) * low_bits)
    return st


def _cpu_info():
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        import psutil
        phys = psutil.cpu_count(logical=False)
    except Exception:  # noqa: BLE001
        phys = None
    return {"model": model, "logical_cpus": os.cpu_count(), "physical_cores": phys}


class Resident:
    """One config's device-resident product (inputs already in HBM, output
    left in HBM) through tc_stage_inputs + tc_execute."""

    def __init__(self, ctx, config):
        import ctypes
        from paper_1612_05778_b200 import _lib
        from paper_1612_05778_b200.params import plan_gpu
        from paper_1612_05778_b200.zpoly import output_bit_width
        self.ctx, self.lib, self.h = ctx, ctx.lib, ctx.handle
        self.config = config
        (aw, ab), (bw, bb) = workloads.make_inputs(config)
        self.aw, self.ab, self.bw, self.bb = aw, ab, bw, bb
        self.da, self.db = aw.shape[0], bw.shape[0]
        self.rows = self.da + self.db - 1
        lib, h = self.lib, self.h
        self.d_a, self.d_b = self._alloc(aw.nbytes), self._alloc(bw.nbytes)
        _lib.check(lib.tc_memcpy(h, self.d_a, _lib.ptr(aw), aw.nbytes, 1), "H2D")
        _lib.check(lib.tc_memcpy(h, self.d_b, _lib.ptr(bw), bw.nbytes, 1), "H2D")
        info = _lib.TcInputInfo()
        _lib.check(lib.tc_stage_inputs(h, self.d_a, self.da, aw.shape[1], self.d_b, self.db, bw.shape[1], 1,
                                       ctypes.byref(info)), "stage")
        self.n_in = max(info.n_in_a, info.n_in_b)
        self.out_bits = output_bit_width(max(self.da, self.db), self.n_in)
        self.out_cw = -(-self.out_bits // 64)
        self.d_out = self._alloc(self.rows * self.out_cw * 8)
        # the plan of these shapes, made once from the measured widths (as a
        # resident caller re-running one shape would); every timed step still
        # runs the device width scans, the whole product and the error checks
        self.plan = plan_gpu(max(self.da, self.db), min(self.da, self.db), self.n_in)
        self.c_plan = _lib.make_plan(self.plan)
        self.out_gbit = self.rows * self.out_bits / 1e9

    def _alloc(self, nbytes):
        import ctypes
        from paper_1612_05778_b200 import _lib
        p = ctypes.c_void_p()
        _lib.check(self.lib.tc_device_alloc(self.h, nbytes, ctypes.byref(p)), "tc_device_alloc")
        return p

    def free(self):
        for p in (self.d_a, self.d_b, self.d_out):
            self.lib.tc_device_free(self.h, p)

    def step(self):
        import ctypes
        from paper_1612_05778_b200 import _lib
        lib, h = self.lib, self.h
        _lib.check(lib.tc_stage_inputs(h, self.d_a, self.da, self.aw.shape[1], self.d_b, self.db,
                                       self.bw.shape[1], 1, None), "stage")
        err = ctypes.c_int64(-1)
        rc = lib.tc_execute(h, ctypes.byref(self.c_plan), self.ab, self.bb, self.d_out, self.rows, self.out_cw, 1,
                            None, ctypes.byref(err))
        _lib.check(rc, "tc_execute")
        if err.value >= 0:
            raise SystemExit(f"bench: corrupted convolution reported at {err.value}")

    def verify(self):
        """Correctness gate (like tc/bench.py:110-125): no timing without parity."""
        from paper_1612_05778_b200 import _lib
        self.step()
        host_out = np.empty((self.rows, self.out_cw), dtype=np.uint64)
        _lib.check(self.lib.tc_memcpy(self.h, _lib.ptr(host_out), self.d_out, host_out.nbytes, 2), "D2H")
        golden = json.load(open(os.path.join(ROOT, "tests", "golden", "configs.json"))).get(self.config)
        if not golden:
            return None
        ok = workloads.words_sha256(host_out) == golden["out_sha256"] and self.out_bits == golden["out_bits"]
        if not ok:
            raise SystemExit(f"bench: product mismatch vs the reference hash for {self.config}")
        return True

    def timed(self):
        """CUDA-event time (ms) of one step on the library's stream, L2 flushed before."""
        import ctypes
        from paper_1612_05778_b200 import _lib
        lib, h = self.lib, self.h
        _lib.check(lib.tc_flush_l2(h), "flush")
        _lib.check(lib.tc_record_event(h, 0), "event")
        self.step()
        _lib.check(lib.tc_record_event(h, 1), "event")
        ms = ctypes.c_float()
        _lib.check(lib.tc_event_elapsed(h, 0, 1, ctypes.byref(ms)), "elapsed")
        return ms.value

    def stage_profile(self):
        """Per-stage event times of one more step (same kernels, enqueued
        directly with stage events instead of the captured graph)."""
        import ctypes
        from paper_1612_05778_b200 import _lib
        _lib.check(self.lib.tc_set_profiling(self.h, 1), "profiling")
        self.timed()
        _lib.check(self.lib.tc_set_profiling(self.h, 0), "profiling")
        prof = (ctypes.c_double * 8)()
        self.lib.tc_last_profile(self.h, prof, None)
        return list(prof)[:5]


E2E_STEPS = []          # per-call wall times (ms) of every e2e_loop, in call order


def e2e_loop(ctx, aw, ab, bw, bb, steps, warmup, pinned):
    """multiply(MulRequest(a, b)) end to end from host arrays: H2D of both
    operands, every kernel and the D2H of the product inside the timed region
    (wall clock around the synchronous call).  pinned=False: the plain
    (pageable) numpy arrays a drop-in caller holds."""
    import paper_1612_05778_b200 as tc
    from paper_1612_05778_b200 import _lib
    if pinned:
        pa = _lib.pinned.empty(aw.shape, np.uint64)
        pb = _lib.pinned.empty(bw.shape, np.uint64)
        pa[...] = aw
        pb[...] = bw
    else:
        pa, pb = aw, bw
    A = tc.IntPolynomial._trusted(pa, ab)
    B = tc.IntPolynomial._trusted(pb, bb)
    lib, h = ctx.lib, ctx.handle
    for _ in range(warmup):
        _lib.check(lib.tc_flush_l2(h), "flush")
        lib.tc_synchronize(h)
        tc.multiply(tc.MulRequest(A, B))
    ts = []
    for _ in range(steps):
        _lib.check(lib.tc_flush_l2(h), "flush")
        lib.tc_synchronize(h)
        t0 = time.perf_counter()
        prod = tc.multiply(tc.MulRequest(A, B))
        ts.append(time.perf_counter() - t0)
        del prod
    E2E_STEPS.append([round(1e3 * t, 2) for t in ts])
    return float(np.sum(ts))


def run_ours(args, rank, world, local):
    import ctypes
    from paper_1612_05778_b200 import _lib
    from paper_1612_05778_b200.params import pass_layout

    ctx = _lib.context(local)
    lib, h = ctx.lib, ctx.handle
    R = Resident(ctx, args.config)
    verified = R.verify()

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        R.timed()
    _barrier(world)
    l0 = ctx.launches()
    times = [R.timed() for _ in range(args.steps)]
    launches = ctx.launches() - l0
    prof = R.stage_profile()
    dev_ms_max = _max_over_ranks(float(np.sum(times)), world)

    # end to end through the public API: plain numpy inputs (the headline)
    # and pinned ones
    e2e_s = _max_over_ranks(e2e_loop(ctx, R.aw, R.ab, R.bw, R.bb, args.steps, args.warmup, pinned=False), world)
    e2e_pin_s = _max_over_ranks(e2e_loop(ctx, R.aw, R.ab, R.bw, R.bb, args.steps, args.warmup, pinned=True), world)

    out_gbit = R.out_gbit
    value = world * args.steps * out_gbit / (dev_ms_max / 1e3)
    e2e_value = world * args.steps * out_gbit / e2e_s
    e2e_pin_value = world * args.steps * out_gbit / e2e_pin_s

    # the other BASELINE configs: device-resident and end-to-end figures
    extras = {}
    plan = R.plan
    aw_nbytes, bw_nbytes, rows, out_cw = R.aw.nbytes, R.bw.nbytes, R.rows, R.out_cw
    R.free()
    for cfg in [c for c in args.extra.split(",") if c and c != args.config]:
        X = Resident(ctx, cfg)
        xv = X.verify()
        for _ in range(3):
            X.timed()
        xs = [X.timed() for _ in range(args.steps)]
        xe = e2e_loop(ctx, X.aw, X.ab, X.bw, X.bb, args.steps, 2, pinned=False)
        xp = e2e_loop(ctx, X.aw, X.ab, X.bw, X.bb, args.steps, 2, pinned=True)
        extras[cfg] = {"value": round(args.steps * X.out_gbit / (float(np.sum(xs)) / 1e3), 3), "unit": "Gbit/s",
                       "ms_per_step": round(float(np.mean(xs)), 4),
                       "e2e": {"value": round(args.steps * X.out_gbit / xe, 3), "ms_per_step": round(1e3 * xe / args.steps, 4)},
                       "e2e_pinned": {"value": round(args.steps * X.out_gbit / xp, 3),
                                      "ms_per_step": round(1e3 * xp / args.steps, 4)},
                       "plan": X.plan.describe(), "verified_vs_reference_sha256": xv}
        X.free()
    clock_info = clocks.stop()
    clock_info["window"] = "the warm-up, timed and e2e loops of every config"

    # roofline: every stage's fractions, the longest stage named
    peaks = _peaks()
    bfly_peak = ctypes.c_double()
    mont_peak = ctypes.c_double()
    lib.tc_int_peak(h, ctypes.byref(bfly_peak), ctypes.byref(mont_peak))
    model = stage_model(plan, R.da, R.db, R.aw.shape[1], R.bw.shape[1], out_cw)
    names = ["convert", "ntt_forward", "pointwise", "ntt_inverse", "recover"]
    stage_ms = dict(zip(names, prof))
    stages = {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    for n in names:
        ms = stage_ms[n]
        m = model[n]
        gbs = m["bytes"] / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
        gbf = m["bfly"] / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
        stages[n] = dict(ms=round(ms, 4), GBps=round(gbs, 1), hbm_frac=round(gbs / hbm_peak, 3),
                         Gbfly_s=round(gbf, 1),
                         int_frac=round(gbf / (bfly_peak.value / 1e9), 3) if bfly_peak.value else None,
                         share_of_step=round(ms / max(sum(stage_ms.values()), 1e-9), 3))
    dom = max(names, key=lambda n: stage_ms[n])
    ds = stages[dom]
    if (ds["int_frac"] or 0) >= ds["hbm_frac"]:
        roof = {"bound": "int", "achieved": ds["Gbfly_s"], "peak": round(bfly_peak.value / 1e9, 1),
                "unit": "Gbutterfly/s", "frac": ds["int_frac"]}
    else:
        roof = {"bound": "hbm", "achieved": ds["GBps"], "peak": hbm_peak, "unit": "GB/s",
                "frac": ds["hbm_frac"]}
    # DRAM traffic per launch of the dominant stage's kernel, from the committed
    # ncu --set full capture of this config
    traffic, tsrc = None, None
    for tf in ("r2_traffic.json", "r1_traffic.json"):
        try:
            tj = json.load(open(os.path.join(ROOT, "profiles", tf))).get(args.config)
            if tj and dom in tj["stages"]:
                ls = tj["stages"][dom]
                traffic = round(sum(x["dram_bytes"] for x in ls) / len(ls))
                tsrc = f"{tj['source']}: {ls[0]['kernel']}, {len(ls)} launch(es) per product"
                break
        except (OSError, ValueError, KeyError):
            pass
    nh = len(pass_layout(plan.L.bit_length() - 1, plan.s_y.bit_length() - 1, plan.P)[1])
    nlaunch = {"convert": 2, "ntt_forward": max(1, 2 * nh - 1), "ntt_inverse": max(1, nh - 1)}.get(dom, 1)
    ncu = None
    for nf in ("r2_ncu_metrics.json", "r1_ncu_metrics.json"):
        try:
            nj = json.load(open(os.path.join(ROOT, "profiles", nf))).get(args.config)
            if nj:
                ncu = nj["kernels"]
                break
        except (OSError, ValueError, KeyError):
            pass
    mm = canonical_modmuls(args.config)
    roof.update({"kernel": dom, "traffic": traffic, "traffic_source": tsrc, "ncu": ncu,
                 "algorithmic_bytes_per_launch": int(model[dom]["bytes"] // nlaunch),
                 "peak_source": "hbm: MEASURED_PEAKS.json hbm_gbs (measured); int: tc_int_peak "
                                "register-only butterfly chain, measured live",
                 "stages": stages,
                 "canonical": {"modmuls_per_product": mm, "unit": "64-bit modmul/s (SURVEY 8(d) MM, reference plan)",
                               "effective_rate": round(mm / (dev_ms_max / args.steps / 1e3), 1),
                               "note": "the reference's own work count at P = 2 over the device-resident time; "
                                       "this build does different (32-bit, pruned, fewer-prime) work"}})

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "Gbit/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dev_ms_max / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded PCG64, BASELINE.md section 4 recipe)",
        "config": {"workload": f"{args.config}: {workloads.CONFIGS[args.config].text}",
                   "d": max(R.da, R.db), "N": workloads.CONFIGS[args.config].N,
                   "rows": rows, "out_bits": R.out_bits,
                   "plan": plan.describe(), "parallelism": f"replicas x{world}",
                   "l2": "flushed (256 MiB memset) before every timed step (device-resident and e2e)",
                   "timed_step": "device width scans + tc_execute (all kernels, error flags read back) "
                                 "with the plan made once for these shapes",
                   "verified_vs_reference_sha256": verified},
        "e2e": {"value": round(e2e_value, 3), "unit": "Gbit/s",
                "ms_per_step": round(1e3 * e2e_s / args.steps, 4),
                "h2d_bytes_per_step": int(aw_nbytes + bw_nbytes),
                "d2h_bytes_per_step": int(rows * out_cw * 8),
                "ms_per_step_median": round(float(np.median(E2E_STEPS[0])), 2), "steps_ms": E2E_STEPS[0],
                "api": "paper_1612_05778_b200.multiply(MulRequest) on plain (pageable) numpy arrays"},
        "e2e_pinned": {"value": round(e2e_pin_value, 3), "unit": "Gbit/s",
                       "ms_per_step": round(1e3 * e2e_pin_s / args.steps, 4),
                       "ms_per_step_median": round(float(np.median(E2E_STEPS[1])), 2), "steps_ms": E2E_STEPS[1],
                       "api": "the same call on page-locked host arrays"},
        "roofline": roof,
        "gpu_launches": int(launches),
        "int_peak": {"butterflies_per_s": bfly_peak.value, "montmul_per_s": mont_peak.value},
        "clocks": clock_info,
        "other_configs": extras,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, R.aw, R.ab, R.bw, R.bb, out_gbit)
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_sharded(args, rank, world, local):
    """N > 1 (torchrun): ONE product over all ranks (strong scaling):
    shard.DistributedMultiplier, the prime split while N <= P (every rank
    transforms its primes, one NCCL exchange of finished residues by row
    tiles), else the row split (compact inputs, two transposes).  Each rank
    ends with its product rows; the device time stops there, the e2e time
    includes every rank's upload of what it reads and its strided download of
    its rows into its host buffer (no gather)."""
    import torch
    import paper_1612_05778_b200 as tc
    from paper_1612_05778_b200 import _lib, shard
    local = local if torch.cuda.device_count() > local else 0   # (single-GPU smoke of this path)
    torch.cuda.set_device(local)
    (aw, ab), (bw, bb) = workloads.make_inputs(args.config)
    pa = _lib.pinned.empty(aw.shape, np.uint64)
    pb = _lib.pinned.empty(bw.shape, np.uint64)
    pa[...] = aw
    pb[...] = bw
    A, B = tc.IntPolynomial._trusted(pa, ab), tc.IntPolynomial._trusted(pb, bb)
    dm = shard.DistributedMultiplier(local)
    rows = aw.shape[0] + bw.shape[0] - 1
    # correctness gate on rank 0
    out, plan = dm.multiply(A, B)
    mode = shard.choose_mode(plan, world)
    verified = None
    if rank == 0:
        golden = json.load(open(os.path.join(ROOT, "tests", "golden", "configs.json"))).get(args.config)
        if golden:
            verified = workloads.words_sha256(out.words) == golden["out_sha256"]
            if not verified:
                raise SystemExit(f"bench: sharded product mismatch vs the reference hash for {args.config}")
        out_bits = out.bit_width
    else:
        out_bits = 0
    del out
    clocks = ClockSampler(local)
    clocks.start()

    def timed(fn):
        _lib.check(dm.ctx.lib.tc_flush_l2(dm.ctx.handle), "flush")     # every rank, before every timed step
        dm._sync()
        torch.cuda.synchronize()
        _barrier(world)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        fn()
        torch.cuda.synchronize()
        dm._sync()
        ev1.record()
        ev1.synchronize()
        return ev0.elapsed_time(ev1)

    resident = mode == "primes"
    if resident:
        dm.upload(A, B)
    for _ in range(args.warmup):
        timed(lambda: dm.multiply(A, B, to_host="device", resident=resident))
    l0 = dm.ctx.launches()
    dev = [timed(lambda: dm.multiply(A, B, to_host="device", resident=resident)) for _ in range(args.steps)]
    launches = dm.ctx.launches() - l0
    e2e = [timed(lambda: dm.multiply(A, B, to_host="local")) for _ in range(args.steps)]
    clock_info = clocks.stop()
    dev_ms = _max_over_ranks(float(np.sum(dev)), world)
    e2e_ms = _max_over_ranks(float(np.sum(e2e)), world)
    out_bits = int(_max_over_ranks(float(out_bits), world))
    out_gbit = rows * out_bits / 1e9
    if rank != 0:
        return
    out_cw = -(-out_bits // 64)
    line = {
        "metric": METRIC, "value": round(args.steps * out_gbit / (dev_ms / 1e3), 3), "unit": "Gbit/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dev_ms / args.steps, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded PCG64, BASELINE.md section 4 recipe)",
        "config": {"workload": f"{args.config}: {workloads.CONFIGS[args.config].text}",
                   "plan": plan.describe(),
                   "parallelism": f"sharded x{world}, {mode} split ({torch.distributed.get_backend()} exchanges)",
                   "l2": "flushed (256 MiB memset) on every rank before every timed step",
                   "timed_step": "device: every rank's product rows finished on its GPU"
                                 + (" (operands resident)" if resident else " (rank's share uploaded)"),
                   "verified_vs_reference_sha256": verified},
        "e2e": {"value": round(args.steps * out_gbit / (e2e_ms / 1e3), 3), "unit": "Gbit/s",
                "ms_per_step": round(e2e_ms / args.steps, 4),
                "h2d_bytes_per_step": int((aw.nbytes + bw.nbytes) * (world if mode == "primes" else 1)),
                "d2h_bytes_per_step": int(rows * out_cw * 8),
                "api": "shard.DistributedMultiplier.multiply(to_host='local') on pinned host arrays: each rank "
                       "uploads what it reads and downloads its own rows (no gather)"},
        "gpu_launches": int(launches), "clocks": clock_info,
        "roofline": None,
    }
    print(json.dumps(line), flush=True)


def canonical_modmuls(config):
    """MM = 2P [3 (S/2) log2 S + 2S] + 2P d K of the
    reference plan (P = 2) of this config: the reference's own work count."""
    from oracle import port   # noqa: F401  (planning only: the reference plan's shape)
    c = workloads.CONFIGS[config]
    n_in = 64 if c.kind == "int64" else c.N + 1
    pl = port.plan_from_shape(c.d, n_in, 2)
    P, S = len(pl.primes), pl.s_y * pl.K
    return 2 * P * (3 * (S // 2) * (S.bit_length() - 1) + 2 * S) + 2 * P * c.d * pl.K


def cpu_baseline(config, aw, ab, bw, bb, out_gbit):
    """The reference's algorithm on this host's cores (oracle/, a C
    restatement of the reference's numba kernels with its 63-bit primes and
    its own plan; the Python reference cannot travel to this box): one full
    product on every host thread with its stage split (the reference's
    StageTimings layout), and a one-thread sample -- the first 4096
    coefficients of each operand, coefficient width unchanged -- sized to
    ~10 s (a full one-thread C3 product takes minutes)."""
    from oracle import port
    threads = os.cpu_count() or 1
    port.multiply_words(aw[:64], ab, bw[:64], bb, threads=threads)   # warm tables / pages
    t0 = time.perf_counter()
    _, _, st = port.multiply_words(aw, ab, bw, bb, threads=threads, stats=True)
    t = time.perf_counter() - t0
    stages = {k: round(v * 1e3, 1) for k, v in st.items()}
    rows = aw.shape[0] + bw.shape[0] - 1
    sub = min(4096, aw.shape[0], bw.shape[0])
    if sub < aw.shape[0]:
        sa, sb = aw[:sub], bw[:sub]
    else:
        sa, sb = aw, bw
    t1 = time.perf_counter()
    _, sbits = port.multiply_words(sa, ab, sb, bb, threads=1)
    t1 = time.perf_counter() - t1
    sub_gbit = (2 * sa.shape[0] - 1) * sbits / 1e9
    return {"value": round(out_gbit / t, 4), "unit": "Gbit/s", "cores": threads, "kind": "port",
            "ms_per_product": round(t * 1e3, 1), "stage_ms": stages,
            "numeric_only_ms": round(t * 1e3, 1),
            "numeric_only_note": "the C restatement has no Python-int scans (tc/params.py:290-293, "
                                 "tc/zpoly.py:45-48,103-114), so total = numeric-only",
            "cpu": _cpu_info(),
            "sample": f"1 full {config} product (reference algorithm: 63-bit primes, P=2, reference plan), "
                      f"OpenMP over all {threads} host threads",
            "w1": {"value": round(sub_gbit / t1, 4), "unit": "Gbit/s", "cores": 1, "ms": round(t1 * 1e3, 1),
                   "sample": f"first {sa.shape[0]} coefficients of each {config} operand (same width), 1 thread"}}


def run_reference(args, rank, world):
    if rank != 0:
        return
    from oracle import port
    from paper_1612_05778_b200 import workloads
    (aw, ab), (bw, bb) = workloads.make_inputs(args.config)
    threads = os.cpu_count() or 1
    # each step is one FULL product of the workload (C3: ~24 s on the box's 16
    # cores, so 20 steps take ~8 minutes).  A smaller sample is not
    # representative: measured on the box, the first 16384 coefficients of C3
    # run at 0.60 Gbit/s against 0.73 for the whole product (the port's fixed
    # per-product costs), which would inflate the GPU/CPU ratio.
    # TC_REF_SAMPLE_D=n (quick local runs only) multiplies the first n.
    full_d = aw.shape[0]
    sample_d = int(os.environ.get("TC_REF_SAMPLE_D", "0"))
    if 0 < sample_d < aw.shape[0]:
        aw, bw = aw[:sample_d], bw[:sample_d]
    rows = aw.shape[0] + bw.shape[0] - 1
    out_bits = port.product_bit_width(aw, bw)
    out_gbit = rows * out_bits / 1e9
    # warm-up: the C restatement has no JIT; one product of the first 1024
    # coefficients pages in its code and tables (full warm-up products would
    # only lengthen the run: a C3 product takes seconds)
    if args.warmup:
        port.multiply_words(aw[:1024], ab, bw[:1024], bb, threads=threads)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        port.multiply_words(aw, ab, bw, bb, threads=threads)
        ts.append(time.perf_counter() - t0)
    tot = float(np.sum(ts))
    value = args.steps * out_gbit / tot
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "Gbit/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * tot / args.steps, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded PCG64, BASELINE.md section 4 recipe)",
        "config": {"workload": f"{args.config}: {workloads.CONFIGS[args.config].text}",
                   "parallelism": "CPU, all host threads"},
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 4), "unit": "Gbit/s", "cores": threads, "kind": "port",
                         "sample": (f"{args.steps} full {args.config} products" if aw.shape[0] == full_d else
                                    f"{args.steps} products of the first {aw.shape[0]} of the {full_d} coefficients "
                                    f"of each {args.config} operand (TC_REF_SAMPLE_D)") + ", oracle/ C restatement "
                                   f"of the reference kernels (the reference is pure Python/numba "
                                   f"and is not present on the GPU box); warm-up: one product of "
                                   f"the first 1024 coefficients",
                         "cpu": _cpu_info()},
        "e2e": {"value": round(value, 4), "unit": "Gbit/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


_dist_ready = False


def _init_dist(world, local):
    global _dist_ready
    if world > 1 and not _dist_ready:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local if torch.cuda.device_count() > local else 0)
        # TC_DIST_BACKEND=gloo only to exercise the N > 1 code path on a single GPU
        dist.init_process_group(os.environ.get("TC_DIST_BACKEND", "nccl"))
        _dist_ready = True


def _barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def _max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--extra", default="C1,C2,C4,C5",
                    help="other BASELINE configs measured beside the headline (other_configs)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    rank, world, local = _dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    _init_dist(world, local)
    if world > 1:
        run_sharded(args, rank, world, local)
    else:
        run_ours(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
