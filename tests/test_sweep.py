"""The correctness-gated sweep (paper_1612_05778_b200/sweep.py, SURVEY.md
section 8(f) item 4) against the reference's own sweep (tests/golden/sweep.json,
made by tests/golden/make_sweep_golden.py from tc/bench.py)."""
import csv
import hashlib
import random

import numpy as np
import pytest

from conftest import load_golden

import paper_1612_05778_b200 as tc
from paper_1612_05778_b200 import sweep


def _sha(w):
    return hashlib.sha256(np.ascontiguousarray(w).tobytes()).hexdigest()


def test_generated_inputs_and_comparators_match_reference():
    meta, _ = load_golden("sweep")
    for pt in meta["points"]:
        d, N, seed = pt["d"], pt["N"], pt["seed"]
        a = sweep.generate_random_dense(d, N, sweep._input_seed(seed, d, N, 0))
        b = sweep.generate_random_dense(d, N, sweep._input_seed(seed, d, N, 1))
        assert _sha(a.words) == pt["a_sha"] and _sha(b.words) == pt["b_sha"] and a.bit_width == pt["a_bits"]
        k = sweep.kronecker_multiply(a, b)
        assert k.bit_width == pt["out_bits"] and list(k.words.shape) == pt["out_shape"]
        assert _sha(k.words) == pt["out_sha"], pt
        if d <= 100:
            assert sweep.schoolbook_multiply(a, b) == k


def test_kronecker_matches_reference_golden_products():
    meta, arr = load_golden("products")
    for m in meta:
        if m["error"]:
            continue
        a = tc.IntPolynomial(arr[f"c{m['id']}_a"], m["a_bits"])
        b = tc.IntPolynomial(arr[f"c{m['id']}_b"], m["b_bits"])
        if a.is_zero() or b.is_zero():
            continue
        k = sweep.kronecker_multiply(a, b)
        assert k.bit_width == m["out_bits"] and np.array_equal(k.words, arr[f"c{m['id']}_out"]), m["id"]


def test_kronecker_extremes_and_unbalanced():
    rng = random.Random(5)
    for _ in range(30):
        da, db = rng.randint(1, 40), rng.randint(1, 40)
        na, nb = rng.randint(1, 300), rng.randint(1, 300)
        ca = [rng.choice([-(1 << (na - 1)), (1 << (na - 1)) - 1, 0, -1, rng.randint(-(1 << (na - 1)), 0)])
              for _ in range(da)]
        cb = [rng.choice([-(1 << (nb - 1)), (1 << (nb - 1)) - 1, 0, 1, rng.randint(0, (1 << (nb - 1)) - 1)])
              for _ in range(db)]
        if not any(ca) or not any(cb):
            continue
        a = tc.IntPolynomial.from_coefficients(ca, bit_width=na)
        b = tc.IntPolynomial.from_coefficients(cb, bit_width=nb)
        assert sweep.kronecker_multiply(a, b) == sweep.schoolbook_multiply(a, b)
    with pytest.raises(tc.EmptyInputError):
        sweep.kronecker_multiply(tc.IntPolynomial.from_coefficients([0]), tc.IntPolynomial.from_coefficients([1]))


def test_sweep_grammar_and_config_validation():
    assert sweep.parse_sweep("d=N:2^9..2^11") == [(512, 512), (1024, 1024), (2048, 2048)]
    assert sweep.parse_sweep("d=N:8,16") == [(8, 8), (16, 16)]
    assert sweep.parse_sweep("512x512,1024x2^8") == [(512, 512), (1024, 256)]
    for bad in ("d=N:8..4", "512", "d=N:0..4"):
        with pytest.raises(ValueError):
            sweep.parse_sweep(bad)
    with pytest.raises(ValueError):
        sweep.BenchConfig(sweep=[])
    with pytest.raises(ValueError):
        sweep.BenchConfig(sweep=[(4, 4)], trials=0)
    with pytest.raises(ValueError):
        sweep.BenchConfig(sweep=[(4, 4)], algorithms=("fft",))
    assert sweep.main(["--sweep", "bad"]) == 2
    assert sweep.main(["--algorithms", "fft"]) == 2


def test_gate_refuses_disagreeing_algorithms(tmp_path, monkeypatch):
    """A wrong-but-fast algorithm stops the sweep before any timing is written."""
    def wrong(a, b):
        p = sweep.schoolbook_multiply(a, b)
        w = p.words.copy()
        w[1, 0] ^= np.uint64(2)
        return tc.IntPolynomial._trusted(w, p.bit_width)
    monkeypatch.setattr(sweep, "kronecker_multiply", wrong)
    cfg = sweep.BenchConfig(sweep=[(8, 8)], algorithms=("schoolbook", "kronecker"), trials=1,
                            output_path=tmp_path / "r.csv")
    with pytest.raises(tc.BenchMismatchError) as ei:
        sweep.run_benchmark(cfg)
    assert "kronecker disagrees with schoolbook at degree 1" in ei.value.report
    assert not (tmp_path / "r.csv").exists()


def test_cpu_sweep_writes_reference_csv(tmp_path):
    meta, _ = load_golden("sweep")
    out = tmp_path / "r.csv"
    rows = sweep.run_benchmark(sweep.BenchConfig(sweep=[(8, 8), (16, 40)], algorithms=("kronecker", "schoolbook"),
                                                 trials=2, output_path=out))
    assert len(rows) == 4 and all(r["correctness_ok"] for r in rows)
    header = open(out).readline().strip().split(",")
    assert header == meta["csv_header"]


@pytest.mark.gpu
def test_gpu_sweep_gated_against_comparators(tmp_path):
    out = tmp_path / "r.csv"
    rc = sweep.main(["--sweep", "d=N:2^5..2^9", "--algorithms", "gpu,kronecker,cvl", "--trials", "2",
                     "--workers", "1,2", "--out", str(out)])
    assert rc == 0
    rows = list(csv.DictReader(open(out)))
    assert len(rows) == 5 * 5 and {r["algorithm"] for r in rows} == {"gpu", "kronecker", "cvl"}
    g = [r for r in rows if r["algorithm"] == "gpu"]
    assert all(r["correctness_ok"] == "True" and r["convert_ms"] != "" for r in g)


@pytest.mark.gpu
def test_gpu_products_on_reference_sweep_points():
    meta, _ = load_golden("sweep")
    for pt in meta["points"]:
        d, N, seed = pt["d"], pt["N"], pt["seed"]
        a = sweep.generate_random_dense(d, N, sweep._input_seed(seed, d, N, 0))
        b = sweep.generate_random_dense(d, N, sweep._input_seed(seed, d, N, 1))
        p = tc.multiply(tc.MulRequest(a, b))
        assert p.bit_width == pt["out_bits"] and _sha(p.words) == pt["out_sha"], pt
