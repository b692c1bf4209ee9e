"""GPU parity of the shapes beyond one 2-D transform: the Kronecker reductions
(csrc/tc_split.cuh) and the long y transforms of the high-valuation primes,
against the CPU oracle (oracle/, the reference's algorithm restated) and,
where the oracle would take minutes, the size-independent evaluation
property c(r) = a(r) b(r) mod q plus exact edge coefficients.  Bit-exact."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1612_05778_b200 as tc  # noqa: E402
from paper_1612_05778_b200.params import SPLIT_COEF, SPLIT_POLY, SplitSpec, plan_gpu  # noqa: E402


def _random_poly(rng, d, nbits, extremes=False):
    lo, hi = -(1 << (nbits - 1)), (1 << (nbits - 1)) - 1
    while True:
        if extremes:
            coeffs = [rng.choice([lo, hi, -1, 0]) for _ in range(d)]
        else:
            coeffs = [rng.randint(lo, hi) for _ in range(d)]
        if any(coeffs):
            return tc.IntPolynomial.from_coefficients(coeffs, bit_width=nbits)


def _random_words(seed, d, nbits):
    """d random nbits-bit two's-complement coefficients as (d, cw) limbs."""
    rng = np.random.default_rng(seed)
    cw = -(-nbits // 64)
    w = rng.integers(0, 2**64 - 1, endpoint=True, size=(d, cw), dtype=np.uint64)
    top = nbits - 64 * (cw - 1)                     # bits used in the top limb
    if top < 64:
        sign = (w[:, -1] >> np.uint64(top - 1)) & np.uint64(1)
        keep = np.uint64((1 << top) - 1)
        w[:, -1] = np.where(sign == 1, w[:, -1] | ~keep, w[:, -1] & keep)
    return w


def _check_eval(oracle, out, aw, bw):
    for q, r in (((1 << 61) - 1, 0x1234567890ABCDE), ((1 << 31) - 1, 987654321)):
        assert oracle.eval_mod(out.words, q, r) == oracle.eval_mod(aw, q, r) * oracle.eval_mod(bw, q, r) % q


def _edge_coefficients(out, a, b):
    """c_0, c_1 and the top two coefficients exactly, with Python ints."""
    A = lambda i: int.from_bytes(a.words[i].tobytes(), "little", signed=True)   # noqa: E731
    B = lambda i: int.from_bytes(b.words[i].tobytes(), "little", signed=True)   # noqa: E731
    C = lambda i: int.from_bytes(out.words[i].tobytes(), "little", signed=True)  # noqa: E731
    da, db = a.words.shape[0], b.words.shape[0]
    rows = da + db - 1
    for k in (0, 1, rows - 2, rows - 1):
        if 0 <= k < rows:
            exp = sum(A(l) * B(k - l) for l in range(max(0, k - db + 1), min(da, k + 1)))
            assert C(k) == exp, k


def test_forced_coef_splits(oracle):
    rng = random.Random(1201)
    cases = [(1, 1, 100, 64), (3, 2, 300, 64), (7, 9, 1000, 128), (40, 33, 777, 192), (5, 1, 64, 64),
             (12, 12, 4097, 1024), (2, 2, 129, 64)]
    for da, db, nbits, bits in cases:
        for extremes in (False, True):
            a = _random_poly(rng, da, nbits, extremes)
            b = _random_poly(rng, db, max(2, nbits - rng.randrange(0, 40)), extremes)
            sp = SplitSpec(SPLIT_COEF, -(-nbits // bits), bits, da + db - 1)
            out, _, plan = tc.multiply_with_plan(tc.MulRequest(a, b), split=sp)
            exp, obits = oracle.multiply_words(a.words, a.bit_width, b.words, b.bit_width)
            assert out.bit_width == obits and np.array_equal(out.words, exp), plan.describe()


def test_forced_poly_splits(oracle):
    rng = random.Random(1202)
    cases = [(10, 10, 20, 1), (33, 17, 64, 4), (100, 100, 65, 16), (300, 250, 200, 64), (64, 3, 500, 8),
             (129, 129, 1, 32), (5, 70, 33, 2)]
    for da, db, nbits, B in cases:
        for extremes in (False, True):
            a = _random_poly(rng, da, nbits, extremes)
            b = _random_poly(rng, db, nbits, extremes)
            dmin = min(da, db)
            bits = 64 * -(-(dmin.bit_length() + 2 * nbits) // 64)
            sp = SplitSpec(SPLIT_POLY, -(-max(da, db) // B), bits, B)
            out, _, plan = tc.multiply_with_plan(tc.MulRequest(a, b), split=sp)
            exp, obits = oracle.multiply_words(a.words, a.bit_width, b.words, b.bit_width)
            assert out.bit_width == obits and np.array_equal(out.words, exp), plan.describe()


def test_planner_chosen_splits_small(oracle):
    # shapes whose direct plan does not fit k_final's tiles (ADVICE: n_in ~ 300k
    # / 500k bits) or needs K > 2^13
    for seed, (d, nbits) in enumerate(((16, 300000), (2, 500000), (3, 1100000))):
        aw, bw = _random_words(seed, d, nbits), _random_words(seed + 50, d, nbits)
        a, b = tc.IntPolynomial(aw, nbits), tc.IntPolynomial(bw, nbits)
        out, _, plan = tc.multiply_with_plan(tc.MulRequest(a, b))
        exp, obits = oracle.multiply_words(aw, nbits, bw, nbits)
        assert out.bit_width == obits and np.array_equal(out.words, exp), plan.describe()


@pytest.mark.parametrize("d,nbits", [(16, (1 << 21) + 1), (2, (1 << 22) + 1)])
def test_wide_coefficients_match_oracle(d, nbits, oracle):
    aw, bw = _random_words(d, d, nbits), _random_words(d + 1, d, nbits)
    a, b = tc.IntPolynomial(aw, nbits), tc.IntPolynomial(bw, nbits)
    out, _, plan = tc.multiply_with_plan(tc.MulRequest(a, b))
    assert plan.split is not None and plan.split.kind == SPLIT_COEF
    exp, obits = oracle.multiply_words(aw, nbits, bw, nbits)
    assert out.bit_width == obits and np.array_equal(out.words, exp), plan.describe()


def test_long_polynomial_direct_matches_oracle(oracle):
    # d = 2^22 + 1: s_y = 2^24, a y transform only the high-valuation primes
    # (998244353, 754974721, ... k >= 24) carry
    d = (1 << 22) + 1
    aw, bw = _random_words(7, d, 64), _random_words(8, d, 64)
    a, b = tc.IntPolynomial(aw, 64), tc.IntPolynomial(bw, 64)
    out, _, plan = tc.multiply_with_plan(tc.MulRequest(a, b))
    assert plan.split is None and plan.s_y == 1 << 24
    exp, obits = oracle.multiply_words(aw, 64, bw, 64)
    assert out.bit_width == obits and np.array_equal(out.words, exp), plan.describe()


@pytest.mark.parametrize("lgd", [23, 24, 25])
def test_long_polynomials_property(lgd, oracle):
    # 2^23: direct (s_y = 2^24); 2^24: direct with the two k >= 25 primes;
    # 2^25: Kronecker block split (no 30-bit prime has 2^26 | p - 1 twice)
    d = 1 << lgd
    aw, bw = _random_words(lgd, d, 64), _random_words(lgd + 1, d - 5, 64)
    a, b = tc.IntPolynomial(aw, 64), tc.IntPolynomial(bw, 64)
    out, _, plan = tc.multiply_with_plan(tc.MulRequest(a, b))
    assert (plan.split is not None) == (lgd >= 25), plan.describe()
    assert out.words.shape[0] == 2 * d - 6
    _check_eval(oracle, out, aw, bw)
    _edge_coefficients(out, a, b)


def test_split_plans_are_chosen_where_expected():
    assert plan_gpu(1 << 25, 1 << 25, 64).split.kind == SPLIT_POLY
    assert plan_gpu(2, 2, (1 << 22) + 1).split.kind == SPLIT_COEF
    assert plan_gpu(8192, 8192, 8193).split is None
