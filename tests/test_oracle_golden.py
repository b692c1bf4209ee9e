"""CPU: pin the oracle (oracle/port.py + oracle/refport.c) to the reference.

Every golden vector was produced by running the reference package itself
(tests/golden/make_golden.py).  The known-answer tests of the reference's own
suite (pkg/tests/test_ntt2d.py:91-122, test_codec.py:24-37,101-109,
test_multiplier.py:32-39,200-207, test_modfield.py:28-41) are restated too.
"""
import json
import os
import random

import numpy as np
import pytest

from conftest import GOLDEN, load_golden


def test_mont_known_answers(oracle):
    rows = json.load(open(os.path.join(GOLDEN, "mont.json")))
    L = oracle.lib()
    for a, bm, p, ninv, got in rows:
        assert L.orc_mont_mul(int(a), int(bm), int(p), int(ninv)) == int(got)


def test_prime_table_matches_reference_rule(oracle):
    tab = oracle.fourier_prime_table()
    assert len(tab) == 184
    assert (tab[0].p, tab[0].q, tab[0].k, tab[0].generator) == (9223372006790004737, 2147483641, 32, 3)
    assert (tab[1].p, tab[1].generator) == (9223371938070528001, 19)
    ref = "/root/reference/pkg/src/twoconv/data/fourier_primes.txt"
    if os.path.exists(ref):   # build container only: byte-for-byte table agreement
        rows = sorted((tuple(map(int, l.split())) for l in open(ref)
                       if l.strip() and not l.startswith("#")), reverse=True)
        assert rows == [(s.p, s.q, s.k, s.generator) for s in tab]


def test_plans_match_reference(oracle):
    for case in json.load(open(os.path.join(GOLDEN, "plans.json"))):
        try:
            pl = oracle.plan_from_shape(case["d"], case["n_min"], case["prime_count"])
        except Exception as ex:
            assert type(ex).__name__ == case.get("error"), case
            continue
        exp = case["plan"]
        got = dict(d=pl.d, N=pl.N, K=pl.K, M=pl.M, s_y=pl.s_y, e=pl.e, f=pl.f,
                   primes=[s.p for s in pl.primes])
        assert got == exp, case


def test_products_match_reference(oracle):
    meta, arr = load_golden("products")
    for m in meta:
        aw, bw = arr[f"c{m['id']}_a"], arr[f"c{m['id']}_b"]
        try:
            out, bits = oracle.multiply_words(aw, m["a_bits"], bw, m["b_bits"], m["prime_count"])
        except oracle.OracleError as ex:
            assert type(ex).__name__ == m["error"], m
            continue
        assert m["error"] is None
        assert bits == m["out_bits"]
        assert np.array_equal(out, arr[f"c{m['id']}_out"]), m


def test_products_match_python_int_oracles(oracle):
    meta, arr = load_golden("products")
    for m in meta[:30]:
        aw, bw = arr[f"c{m['id']}_a"], arr[f"c{m['id']}_b"]
        ca, cb = oracle.coefficients(aw), oracle.coefficients(bw)
        ref = oracle.schoolbook(ca, cb)
        assert oracle.kronecker(ca, cb) == ref
        assert oracle.coefficients(arr[f"c{m['id']}_out"]) == ref


def test_digits_match_reference(oracle):
    meta, arr = load_golden("digits")
    for m in meta:
        words = arr[f"d{m['id']}_in"]
        plan = oracle.MulPlan(d=words.shape[0], N=m["N"], K=m["K"], M=m["M"], s_y=1, primes=(), e=0, f=0)
        if m["error"]:
            with pytest.raises(oracle.EncodingError):
                oracle.digits(words, m["bits"], plan)
            continue
        assert np.array_equal(oracle.digits(words, m["bits"], plan), arr[f"d{m['id']}_digits"]), m


def test_grids_and_cpm_match_reference(oracle):
    meta, arr = load_golden("cpm")
    gmeta, garr = load_golden("grids")
    for m, g in zip(meta, gmeta):
        n = m["id"]
        pl = m["plan"]
        primes = tuple(s for s in oracle.fourier_prime_table() if s.p in pl["primes"])
        primes = tuple(sorted(primes, key=lambda s: pl["primes"].index(s.p)))
        plan = oracle.MulPlan(d=pl["d"], N=pl["N"], K=pl["K"], M=pl["M"], s_y=pl["s_y"],
                              primes=primes, e=pl["e"], f=pl["f"])
        da, db = arr[f"m{n}_a"], arr[f"m{n}_b"]
        cyc = [oracle.convolve(da, db, plan, t, False) for t in range(len(primes))]
        neg = [oracle.convolve(da, db, plan, t, True) for t in range(len(primes))]
        for t in range(len(primes)):
            assert np.array_equal(cyc[t], garr[f"g{n}_{t}_cyc"])
            assert np.array_equal(neg[t], garr[f"g{n}_{t}_neg"])
        rows = 2 * pl["d"] - 1
        assert np.array_equal(oracle.combine_residues(neg, plan, rows), arr[f"m{n}_cp"])
        assert np.array_equal(oracle.combine_residues(cyc, plan, rows), arr[f"m{n}_cm"])


def _poly(oracle, coeffs, bits=None):
    if bits is None:
        bits = max(oracle.twos_complement_width(c) for c in coeffs)
    return oracle.words_from_coefficients(coeffs, bits), bits


def test_known_answers(oracle):
    # pkg/tests/test_multiplier.py:32-39, 200-207
    for ca, cb, exp in (([1], [1], [1]), ([1, 1], [-1, 1], [-1, 0, 1]),
                        ([3 ** 400], [-(5 ** 340)], [-(3 ** 400) * 5 ** 340])):
        (aw, ab), (bw, bb) = _poly(oracle, ca), _poly(oracle, cb)
        out, bits = oracle.multiply_words(aw, ab, bw, bb)
        assert oracle.coefficients(out) == exp
    # pkg/tests/test_codec.py:24-28: digits 5 -> [1, 1], 3 -> [-1, 1]
    plan = oracle.MulPlan(d=1, N=4, K=2, M=2, s_y=1, primes=(), e=0, f=0)
    for v, dg in ((5, [1, 1]), (3, [-1, 1]), (0, [0, 0]), (-8, [0, -2])):
        w, b = _poly(oracle, [v], 4)
        assert list(oracle.digits(w, b, plan)[0]) == dg


def test_cyclic_negacyclic_known_answers(oracle):
    # (1 + 2x)(3 + 4x): cyclic [11, 10], negacyclic [-5, 10] (pkg/tests/test_ntt2d.py:101-117)
    plan = oracle.plan_for(1, 2, 4)
    a = np.array([[1, 2]], dtype=np.int64)
    b = np.array([[3, 4]], dtype=np.int64)
    p = plan.primes[0].p
    lift = lambda r: int(r) - p if int(r) > (p - 1) // 2 else int(r)
    assert [lift(x) for x in oracle.convolve(a, b, plan, 0, False)[0]] == [11, 10]
    assert [lift(x) for x in oracle.convolve(a, b, plan, 0, True)[0]] == [-5, 10]


def test_worker_counts_bitwise_identical(oracle):
    meta, arr = load_golden("products")
    m = meta[-1]
    aw, bw = arr[f"c{m['id']}_a"], arr[f"c{m['id']}_b"]
    outs = [oracle.multiply_words(aw, m["a_bits"], bw, m["b_bits"], threads=t)[0] for t in (1, 2, 8)]
    assert all(np.array_equal(outs[0], o) for o in outs[1:])


@pytest.mark.parametrize("name", ["C1", "C5", "C2"])
def test_full_config_hash(oracle, name):
    from paper_1612_05778_b200 import workloads
    cfg = json.load(open(os.path.join(GOLDEN, "configs.json")))[name]
    (aw, ab), (bw, bb) = workloads.make_inputs(name)
    assert workloads.words_sha256(aw) == cfg["a_sha256"]
    assert workloads.words_sha256(bw) == cfg["b_sha256"]
    out, bits = oracle.multiply_words(aw, ab, bw, bb)
    assert bits == cfg["out_bits"] and list(out.shape) == cfg["out_shape"]
    assert workloads.words_sha256(out) == cfg["out_sha256"]


def test_eval_mod_property(oracle):
    rng = random.Random(5)
    meta, arr = load_golden("products")
    for m in meta[:10]:
        aw, bw, ow = arr[f"c{m['id']}_a"], arr[f"c{m['id']}_b"], arr[f"c{m['id']}_out"]
        q = (1 << 61) - 1
        r = rng.randrange(q)
        assert oracle.eval_mod(ow, q, r) == oracle.eval_mod(aw, q, r) * oracle.eval_mod(bw, q, r) % q
