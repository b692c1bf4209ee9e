#!/usr/bin/env python3
"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py [--configs C1,C2,C4,C5]

Outputs (all small; committed):
  products.npz + products.json  random products incl. extremes, mixed widths,
                                d=1 and prime counts 1/2/3 (tc/multiplier.py:169-176)
  digits.npz   + digits.json    balanced digits / EncodingError rows (tc/codec.py:71-99)
  cpm.npz      + cpm.json       C+ / C- after CRT (tc/multiplier.py:66-100)
  grids.npz    + grids.json     cyclic / negacyclic residue grids (tc/ntt2d.py:128-135)
  plans.json                    build_plan / plan_from_shape results (tc/params.py)
  mont.json                     Montgomery known answers (tc/_kernels.py:52-55)
  configs.json                  SHA-256 of the reference product for the BASELINE
                                configs, with input hashes, bit width and plan
"""

from __future__ import annotations

import argparse
import json
import os
import random
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import twoconv  # noqa: E402  (the reference)
from twoconv import IntPolynomial, MulRequest, multiply, multiply_with_stats  # noqa: E402
from twoconv import _kernels as rk  # noqa: E402
from twoconv.codec import bivariate_representation, DigitMatrix  # noqa: E402
from twoconv.modfield import mont_constants  # noqa: E402
from twoconv.multiplier import _combine_residues  # noqa: E402
from twoconv.ntt2d import cyclic_convolution, negacyclic_convolution  # noqa: E402
from twoconv.params import build_plan, plan_for, plan_from_shape, fourier_prime_table  # noqa: E402
from twoconv.zpoly import product_bit_width  # noqa: E402

from paper_1612_05778_b200 import workloads  # noqa: E402


def _rand_poly(rng, d, nbits, extremes=False):
    lo, hi = -(1 << (nbits - 1)), (1 << (nbits - 1)) - 1
    while True:
        if extremes:
            coeffs = [rng.choice([lo, hi, 0, -1, 1]) for _ in range(d)]
        else:
            coeffs = [rng.randint(lo, hi) for _ in range(d)]
            if rng.random() < 0.4:
                coeffs[rng.randrange(d)] = lo
            if rng.random() < 0.4:
                coeffs[rng.randrange(d)] = hi
        if any(coeffs):
            return IntPolynomial.from_coefficients(coeffs, bit_width=nbits)


def _plan_dict(plan):
    return dict(d=plan.d, N=plan.N, K=plan.K, M=plan.M, s_y=plan.s_y, e=plan.e, f=plan.f,
                primes=[s.p for s in plan.primes])


def gen_products():
    rng = random.Random(0xC0FFEE)
    arrays, meta = {}, []
    cases = []
    for _ in range(70):
        cases.append((rng.randint(1, 64), rng.randint(1, 300), rng.randint(1, 64),
                      rng.randint(1, 300), rng.choice([1, 2, 2, 3]), rng.random() < 0.15))
    cases += [(1, 1, 1, 1, 2, False), (1, 2000, 1, 1500, 2, False), (300, 8, 3, 700, 2, False),
              (200, 64, 200, 64, 3, True), (2, 126, 2, 126, 3, True), (33, 1025, 31, 1025, 2, False)]
    for n, (da, na, db, nb, pc, ext) in enumerate(cases):
        a = _rand_poly(rng, da, na, ext)
        b = _rand_poly(rng, db, nb, ext)
        entry = dict(id=n, a_bits=a.bit_width, b_bits=b.bit_width, prime_count=pc)
        try:
            out = multiply(MulRequest(a, b, prime_count=pc))
            entry.update(out_bits=out.bit_width, error=None)
            arrays[f"c{n}_out"] = out.words
            entry["plan"] = _plan_dict(build_plan(a, b, pc))
        except Exception as ex:  # PrimeCapacityError with one prime, etc.
            entry.update(out_bits=None, error=type(ex).__name__)
        arrays[f"c{n}_a"] = a.words
        arrays[f"c{n}_b"] = b.words
        meta.append(entry)
    np.savez_compressed(os.path.join(HERE, "products.npz"), **arrays)
    json.dump(meta, open(os.path.join(HERE, "products.json"), "w"), indent=1)
    print("products:", len(meta), "cases,", sum(m["error"] is not None for m in meta), "errors")


def gen_digits():
    rng = random.Random(613)
    arrays, meta = {}, []
    n = 0
    # random plans from shape, incl. extremes (pkg/tests/test_codec.py:40-56)
    for _ in range(40):
        d = rng.randint(1, 24)
        n_min = rng.randint(1, 400)
        plan = plan_from_shape(d, n_min)
        poly = _rand_poly(rng, d, n_min)
        # sign-extend / keep width as the reference test does (bit_width = N)
        poly = IntPolynomial.from_coefficients(poly.coefficients(), bit_width=plan.N)
        mat = bivariate_representation(poly, plan)
        arrays[f"d{n}_in"] = poly.words
        arrays[f"d{n}_digits"] = mat.digits
        meta.append(dict(id=n, bits=poly.bit_width, K=plan.K, M=plan.M, N=plan.N, error=None))
        n += 1
    # explicit K, M incl. M up to 63 and narrower/wider input widths (tc/codec.py:59-68)
    for K, M, width in ((2, 2, 3), (4, 3, 12), (8, 5, 40), (2, 63, 126), (4, 63, 200),
                        (16, 33, 528), (32, 17, 300), (128, 9, 1025), (64, 33, 64)):
        plan = plan_for(5, K, M, prime_count=3)
        poly = _rand_poly(rng, 5, min(width, plan.N))
        poly = IntPolynomial.from_coefficients(poly.coefficients(), bit_width=width)
        entry = dict(id=n, bits=poly.bit_width, K=K, M=M, N=plan.N, error=None)
        try:
            mat = bivariate_representation(poly, plan)
            arrays[f"d{n}_digits"] = mat.digits
        except Exception as ex:
            entry["error"] = type(ex).__name__
        arrays[f"d{n}_in"] = poly.words
        meta.append(entry)
        n += 1
    # encoding errors: beyond digit capacity, and beyond the plan width
    for value, bits, K, M in ((7, 4, 2, 2), (100, 8, 2, 2), (5, 4, 2, 2), (-8, 4, 2, 2), (-7, 4, 2, 2),
                              ((1 << 40) - 5, 42, 4, 10)):
        plan = plan_for(1, K, M)
        poly = IntPolynomial.from_coefficients([1, value, 3], bit_width=bits)
        entry = dict(id=n, bits=bits, K=K, M=M, N=plan.N, error=None)
        try:
            mat = bivariate_representation(poly, plan)
            arrays[f"d{n}_digits"] = mat.digits
        except Exception as ex:
            entry["error"] = type(ex).__name__
            entry["message"] = str(ex)
        arrays[f"d{n}_in"] = poly.words
        meta.append(entry)
        n += 1
    np.savez_compressed(os.path.join(HERE, "digits.npz"), **arrays)
    json.dump(meta, open(os.path.join(HERE, "digits.json"), "w"), indent=1)
    print("digits:", len(meta), "cases")


def gen_cpm_and_grids():
    rng = random.Random(23)
    arrays, meta = {}, []
    garrays, gmeta = {}, []
    for n in range(24):
        d = rng.randint(1, 12)
        K = rng.choice([2, 4, 8, 16])
        M = rng.randint(2, 40)
        pc = rng.choice([1, 2, 3])
        try:
            plan = plan_for(d, K, M, prime_count=pc)
        except Exception:
            plan = plan_for(d, K, M, prime_count=3)
            pc = 3
        half = 1 << (M - 1)
        mk = lambda: np.array([[rng.randint(-half, half - 1) for _ in range(K)]
                               for _ in range(d)], dtype=np.int64)
        a = DigitMatrix(d=d, K=K, M=M, digits=mk())
        b = DigitMatrix(d=d, K=K, M=M, digits=mk())
        cyc = [cyclic_convolution(a, b, plan, t) for t in range(len(plan.primes))]
        neg = [negacyclic_convolution(a, b, plan, t) for t in range(len(plan.primes))]
        rows = 2 * d - 1
        cp = _combine_residues(neg, plan, rows, 1)
        cm = _combine_residues(cyc, plan, rows, 1)
        arrays[f"m{n}_a"] = a.digits
        arrays[f"m{n}_b"] = b.digits
        arrays[f"m{n}_cp"] = cp
        arrays[f"m{n}_cm"] = cm
        meta.append(dict(id=n, d=d, K=K, M=M, prime_count=pc, plan=_plan_dict(plan)))
        for t in range(len(plan.primes)):
            garrays[f"g{n}_{t}_cyc"] = cyc[t].data
            garrays[f"g{n}_{t}_neg"] = neg[t].data
        gmeta.append(dict(id=n, d=d, K=K, M=M, plan=_plan_dict(plan)))
    np.savez_compressed(os.path.join(HERE, "cpm.npz"), **arrays)
    json.dump(meta, open(os.path.join(HERE, "cpm.json"), "w"), indent=1)
    np.savez_compressed(os.path.join(HERE, "grids.npz"), **garrays)
    json.dump(gmeta, open(os.path.join(HERE, "grids.json"), "w"), indent=1)
    print("cpm/grids:", len(meta), "cases")


def gen_plans():
    rng = random.Random(151)
    out = []
    for _ in range(120):
        d = rng.randint(1, 1 << rng.randint(1, 21))
        n_min = rng.randint(1, 1 << rng.randint(1, 19))
        pc = rng.choice([1, 2, 3])
        try:
            out.append(dict(d=d, n_min=n_min, prime_count=pc,
                            plan=_plan_dict(plan_from_shape(d, n_min, pc))))
        except Exception as ex:
            out.append(dict(d=d, n_min=n_min, prime_count=pc, error=type(ex).__name__))
    for d, n_min in ((1024, 1025), (8192, 8193), (65536, 65537), (1 << 20, 64),
                     (256, 262145), (32, 100), (4, 4), (64, 64)):
        for pc in (1, 2, 3):
            try:
                out.append(dict(d=d, n_min=n_min, prime_count=pc,
                                plan=_plan_dict(plan_from_shape(d, n_min, pc))))
            except Exception as ex:
                out.append(dict(d=d, n_min=n_min, prime_count=pc, error=type(ex).__name__))
    json.dump(out, open(os.path.join(HERE, "plans.json"), "w"), indent=1)
    print("plans:", len(out))


def gen_mont():
    rng = random.Random(99)
    out = []
    for spec in fourier_prime_table()[:2]:
        p = spec.p
        r1, ninv = mont_constants(spec)
        for _ in range(200):
            a, b = rng.randrange(p), rng.randrange(p)
            bm = b * r1 % p
            got = int(rk.mont_mul_probe(np.uint64(a), np.uint64(bm), np.uint64(p), np.uint64(ninv)))
            assert got == a * b % p
            out.append([str(a), str(bm), str(p), str(ninv), str(got)])
    json.dump(out, open(os.path.join(HERE, "mont.json"), "w"))
    print("mont:", len(out))


def gen_configs(names):
    path = os.path.join(HERE, "configs.json")
    table = json.load(open(path)) if os.path.exists(path) else {}
    for name in names:
        (aw, ab), (bw, bb) = workloads.make_inputs(name)
        a = IntPolynomial.__new__(IntPolynomial)   # skip the Python-int validation loop
        a.words, a.bit_width = aw, ab
        b = IntPolynomial.__new__(IntPolynomial)
        b.words, b.bit_width = bw, bb
        t0 = time.time()
        out, st = multiply_with_stats(MulRequest(a, b, prime_count=2))
        el = time.time() - t0
        plan = build_plan(a, b, 2)
        table[name] = dict(
            a_sha256=workloads.words_sha256(aw), b_sha256=workloads.words_sha256(bw),
            a_bits=ab, b_bits=bb, out_bits=out.bit_width, out_shape=list(out.words.shape),
            out_sha256=workloads.words_sha256(out.words),
            out_row0_sha256=workloads.words_sha256(out.words[0]),
            out_rowmid_sha256=workloads.words_sha256(out.words[out.words.shape[0] // 2]),
            ref_plan=_plan_dict(plan), ref_seconds=el, ref_workers=st.workers,
            ref_stages={k: getattr(st, k) for k in ("convert", "ntt_forward", "pointwise",
                                                    "ntt_inverse", "crt", "recover", "total")},
        )
        print(name, "out", out.words.shape, out.bit_width, f"{el:.1f}s")
        json.dump(table, open(path, "w"), indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C4,C5")
    ap.add_argument("--skip-small", action="store_true")
    args = ap.parse_args()
    if not args.skip_small:
        gen_products()
        gen_digits()
        gen_cpm_and_grids()
        gen_plans()
        gen_mont()
    if args.configs:
        gen_configs([c for c in args.configs.split(",") if c])


if __name__ == "__main__":
    main()
