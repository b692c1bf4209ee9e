"""CPU: host logic of the product package and the C-ABI library surface."""
import json
import os
import random
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, load_golden

import paper_1612_05778_b200 as tc
from paper_1612_05778_b200 import _lib, params, workloads, zpoly


def test_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "tc_api.h")).read()
    declared = sorted(set(re.findall(r"\b(tc_[a-z0-9_]+)\s*\(", header)))
    assert declared and set(declared) == set(_lib.EXPORTED_SYMBOLS)
    lib = _lib.load()          # loads without a GPU
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.tc_version().startswith(b"tcgpu")


def test_product_path_fails_loudly_without_device():
    lib = _lib.load()
    import ctypes
    h = ctypes.c_void_p()
    rc = lib.tc_ctx_create(-1, ctypes.byref(h))
    if rc == 0:
        lib.tc_ctx_destroy(h)
        pytest.skip("a CUDA device is present")
    with pytest.raises(tc.DeviceError):
        tc.multiply(tc.MulRequest(tc.IntPolynomial.from_coefficients([1]),
                                  tc.IntPolynomial.from_coefficients([2])))


def test_int_polynomial_semantics():
    meta, arr = load_golden("products")
    for m in meta[:20]:
        w = arr[f"c{m['id']}_a"]
        p = tc.IntPolynomial(w, m["a_bits"])
        assert p.max_width() == max(zpoly.twos_complement_width(c) for c in p.coefficients())
        assert p == tc.IntPolynomial.from_coefficients(p.coefficients(), bit_width=m["a_bits"])
    with pytest.raises(ValueError):
        tc.IntPolynomial.from_coefficients([8], bit_width=4)
    with pytest.raises(ValueError):
        tc.IntPolynomial(np.zeros((2, 2), dtype=np.uint64), 64)
    assert tc.IntPolynomial.from_coefficients([-8], bit_width=4).coefficients() == [-8]
    text = tc.format_polynomial(tc.IntPolynomial.from_coefficients([5, -3, 1, 21]))
    assert tc.parse_polynomial(text).coefficients() == [5, -3, 1, 21]


def test_row_widths_match_python_ints():
    rng = random.Random(3)
    for _ in range(20):
        bits = rng.randint(1, 700)
        coeffs = [rng.randint(-(1 << (bits - 1)), (1 << (bits - 1)) - 1) for _ in range(30)]
        coeffs += [0, -1, 1, -(1 << (bits - 1))]
        p = tc.IntPolynomial.from_coefficients(coeffs, bit_width=bits)
        assert list(zpoly.row_widths(p.words)) == [zpoly.twos_complement_width(c) for c in coeffs]


def test_reference_planner_restatement_matches_golden():
    for case in json.load(open(os.path.join(GOLDEN, "plans.json"))):
        try:
            pl = params.plan_from_shape(case["d"], case["n_min"], case["prime_count"])
        except Exception as ex:
            assert type(ex).__name__ == case.get("error"), case
            continue
        got = dict(d=pl.d, N=pl.N, K=pl.K, M=pl.M, s_y=pl.s_y, e=pl.e, f=pl.f,
                   primes=[s.p for s in pl.primes])
        assert got == case["plan"], case


def test_reference_build_plan_matches_golden():
    meta, arr = load_golden("products")
    for m in meta[:40]:
        a = tc.IntPolynomial(arr[f"c{m['id']}_a"], m["a_bits"])
        b = tc.IntPolynomial(arr[f"c{m['id']}_b"], m["b_bits"])
        pl = tc.build_plan(a, b, m["prime_count"])
        assert (pl.K, pl.M, pl.N, pl.e, pl.f) == tuple(m["plan"][k] for k in ("K", "M", "N", "e", "f"))


def test_gpu_prime_table():
    tab = params.gpu_prime_table()
    assert len(tab) >= 100
    assert max(s.k for s in tab) == 26 and sorted(s.p for s in tab if s.k >= 24) == [167772161, 469762049, 754974721]
    for s in tab:
        assert s.p < (1 << 30) and s.k >= 20 and s.p == s.q * (1 << s.k) + 1 and s.q % 2 == 1
        assert params.is_prime_u64(s.p) and params.is_primitive_root(s.generator, s)


def test_gpu_plan_invariants():
    rng = random.Random(11)
    shapes = [(1024, 1025), (8192, 8193), (65536, 65537), (1 << 20, 64), (256, 262145), (1, 1),
              (1, 5000), (3, 2), (2, 1)]
    shapes += [(rng.randint(1, 1 << 16), rng.randint(1, 1 << 15)) for _ in range(60)]
    for d, n_in in shapes:
        dmin = rng.randint(1, d)
        pl = params.plan_gpu(d, dmin, n_in)
        assert pl.K & (pl.K - 1) == 0 and 1 <= pl.K <= params.MAX_K and 2 <= pl.M <= params.MAX_GPU_DIGIT_BITS
        lo, hi = params.balanced_capacity(pl.K, pl.M)
        assert lo <= -(1 << (n_in - 1)) and (1 << (n_in - 1)) - 1 <= hi
        prod = 1
        for s in pl.primes:
            assert (1 << s.k) >= max(pl.s_y, 2 * pl.K)
            prod *= s.p
        assert prod > 2 * pl.coefficient_bound()
        assert pl.s_y >= 2 * d - 1 and pl.s_y & (pl.s_y - 1) == 0


def test_gpu_plans_of_the_baseline_configs():
    # the plans DESIGN.md section 2 documents (each measured against the
    # alternatives on the B200): two-word digits where the grid is large
    exp = {(1024, 1025): (32, 33, 3), (8192, 8193): (128, 65, 5), (65536, 65537): (1024, 65, 6),
           (1 << 20, 64): (1, 64, 5), (256, 262145): (4096, 65, 5)}
    for (d, n_in), (K, M, P) in exp.items():
        pl = params.plan_gpu(d, d, n_in)
        assert (pl.K, pl.M, pl.P) == (K, M, P), pl.describe()
    # the C2 two-word plan is feasible with exactly five 30-bit primes
    pl = params.plan_gpu(8192, 8192, 8193)
    prod = 1
    for s in pl.primes:
        prod *= s.p
    assert prod > 2 * pl.coefficient_bound() and prod // pl.primes[-1].p <= 2 * pl.coefficient_bound()


def test_workload_generators_match_recorded_hashes():
    cfg = json.load(open(os.path.join(GOLDEN, "configs.json")))
    for name in ("C1", "C2", "C5", "C4"):
        if name not in cfg:
            continue
        (aw, ab), (bw, bb) = workloads.make_inputs(name)
        assert workloads.words_sha256(aw) == cfg[name]["a_sha256"]
        assert workloads.words_sha256(bw) == cfg[name]["b_sha256"]
        assert (ab, bb) == (cfg[name]["a_bits"], cfg[name]["b_bits"])
        assert zpoly.fits_width(aw, ab).all() and zpoly.fits_width(bw, bb).all()


def test_signed_generator_distribution():
    (aw, ab), _ = workloads.make_inputs("C1")
    neg = (aw[:, -1] >> np.uint64(63)).astype(bool)
    assert 0.4 < neg.mean() < 0.6
    p = tc.IntPolynomial(aw, ab)
    assert p.max_width() <= 1025
