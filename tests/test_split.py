"""CPU: the Kronecker reductions (params.SplitSpec, csrc/tc_split.cuh) as
integer algebra, and the planner's coverage of every shape the reference
plans (tc/params.py:225-267).

The pack / unpack steps are restated here with Python integers (test
infrastructure): for random operands, unpack(pack(a) * pack(b)) must equal
the schoolbook product exactly, for both reductions and for the plans the
planner emits.  The CUDA kernels themselves are checked bit for bit on the
GPU (tests/test_gpu_split.py)."""
import math
import random

import pytest

from paper_1612_05778_b200 import params
from paper_1612_05778_b200.params import SPLIT_COEF, SPLIT_POLY, SplitSpec


def schoolbook(a, b):
    out = [0] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        if x:
            for j, y in enumerate(b):
                out[i + j] += x * y
    return out


def pack_coef(a, sp: SplitSpec, D: int):
    """Row i + s D = super-digit s of a_i: unsigned Nc-bit chunks, the top one
    signed (k_pack_coef)."""
    rows = [0] * ((sp.n - 1) * D + len(a))
    for i, x in enumerate(a):
        for s in range(sp.n):
            v = x >> (s * sp.bits)                       # arithmetic shift: the sign stays
            rows[i + s * D] = v if s == sp.n - 1 else v & ((1 << sp.bits) - 1)
    return rows


def unpack_coef(ct, sp: SplitSpec, D: int, rows: int):
    """c_i = sum_s c~[i + s D] 2^(s Nc) (k_shift_add)."""
    return [sum(ct[i + s * D] << (s * sp.bits) for s in range(2 * sp.n - 1) if i + s * D < len(ct))
            for i in range(rows)]


def pack_poly(a, sp: SplitSpec):
    """a~_i = sum_t a[t B + i] 2^(t Nz) (k_shift_add)."""
    B = sp.block
    return [sum(a[t * B + i] << (t * sp.bits) for t in range(-(-len(a) // B)) if t * B + i < len(a))
            for i in range(min(B, len(a)))]


def balanced_chunk(x, s, bits):
    """C(s) of x = sum_s C(s) 2^(s bits), C(s) in [-2^(bits-1), 2^(bits-1))."""
    carry = 0
    for t in range(s + 1):
        r = ((x >> (t * bits)) & ((1 << bits) - 1)) + carry
        carry = 1 if r >= 1 << (bits - 1) else 0
        c = r - (carry << bits)
    return c


def unpack_poly(ct, sp: SplitSpec, rows: int):
    """c_(sB+i) = C(s, i) + C(s-1, i+B) (k_unpack_poly)."""
    B = sp.block
    out = []
    for k in range(rows):
        s, i = divmod(k, B)
        v = balanced_chunk(ct[i], s, sp.bits)
        if s >= 1 and i + B < len(ct):
            v += balanced_chunk(ct[i + B], s - 1, sp.bits)
        out.append(v)
    return out


def rand_poly(rng, d, nbits, extremes=False):
    lo, hi = -(1 << (nbits - 1)), (1 << (nbits - 1)) - 1
    return [rng.choice([lo, hi, 0, -1]) if extremes else rng.randint(lo, hi) for _ in range(d)]


@pytest.mark.parametrize("seed", range(6))
def test_coef_split_algebra(seed):
    rng = random.Random(seed)
    for _ in range(8):
        da, db = rng.randint(1, 9), rng.randint(1, 9)
        nbits = rng.randint(2, 700)
        a = rand_poly(rng, da, nbits, extremes=rng.random() < 0.3)
        b = rand_poly(rng, db, nbits, extremes=rng.random() < 0.3)
        bits = 64 * rng.randint(1, 4)
        sp = SplitSpec(SPLIT_COEF, -(-nbits // bits), bits, da + db - 1)
        D = da + db - 1
        pa, pb = pack_coef(a, sp, D), pack_coef(b, sp, D)
        # the inner operands fit the declared inner width Nc + 1
        for v in pa + pb:
            assert -(1 << bits) <= v < (1 << bits)
        assert unpack_coef(schoolbook(pa, pb), sp, D, D) == schoolbook(a, b)


@pytest.mark.parametrize("seed", range(6))
def test_poly_split_algebra(seed):
    rng = random.Random(100 + seed)
    for _ in range(8):
        da, db = rng.randint(1, 60), rng.randint(1, 60)
        nbits = rng.randint(2, 200)
        a = rand_poly(rng, da, nbits, extremes=rng.random() < 0.3)
        b = rand_poly(rng, db, nbits, extremes=rng.random() < 0.3)
        B = 1 << rng.randint(0, 5)
        dmin = min(da, db)
        bits = 64 * -(-(dmin.bit_length() + 2 * nbits) // 64)
        sp = SplitSpec(SPLIT_POLY, -(-max(da, db) // B), bits, B)
        pa, pb = pack_poly(a, sp), pack_poly(b, sp)
        n2 = params.split_inner_shape(sp, max(da, db), dmin, nbits)[2]
        for v in pa + pb:                                  # the declared inner width holds them
            assert -(1 << (n2 - 1)) <= v < (1 << (n2 - 1))
        assert unpack_poly(schoolbook(pa, pb), sp, da + db - 1) == schoolbook(a, b)


def test_min_digit_bits_closed_form():
    for K in (1, 2, 4, 8, 16, 64, 256):
        for n in range(1, 400):
            lo, hi = -(1 << (n - 1)), (1 << (n - 1)) - 1 if n > 1 else 0
            M = params.min_digit_bits(K, n)
            cl, ch = params.balanced_capacity(K, M)
            assert cl <= lo and hi <= ch
            if M > 2:
                cl, ch = params.balanced_capacity(K, M - 1)
                assert not (cl <= lo and hi <= ch)


def _check_plan(pl, d, dmin, n_in):
    assert pl.K & (pl.K - 1) == 0 and 1 <= pl.K <= params.MAX_K and 2 <= pl.M <= params.MAX_GPU_DIGIT_BITS
    prod = math.prod(s.p for s in pl.primes)
    assert prod > 2 * pl.coefficient_bound() and pl.P <= params.MAX_PRIMES
    for s in pl.primes:
        assert (1 << s.k) >= max(pl.s_y, 2 * pl.K) and s.p < (1 << 30)
    assert params.final_tile_bytes(pl.K, pl.s_y, pl.P) <= params.FINAL_SMEM_LIMIT
    assert (pl.s_y * pl.L).bit_length() - 1 <= params.MAX_GRID_BITS
    if pl.split is None:
        assert (pl.d, pl.dmin) == (d, dmin)
        lo, hi = params.balanced_capacity(pl.K, pl.M) if n_in < 5000 else (None, None)
        if lo is not None:
            assert lo <= -(1 << (n_in - 1)) and (1 << (n_in - 1)) - 1 <= hi
        assert pl.K * pl.M >= n_in
    else:
        d2, m2, n2 = params.split_inner_shape(pl.split, d, dmin, n_in)
        assert (pl.d, pl.dmin) == (d2, m2) and pl.K * pl.M >= n2 and pl.outer == (d, dmin, n_in)
        if pl.split.kind == SPLIT_COEF:
            assert pl.split.n * pl.split.bits >= n_in and pl.split.block == d + dmin - 1
        else:
            assert pl.split.bits >= dmin.bit_length() + 2 * n_in and pl.split.n * pl.split.block >= d


def test_plans_cover_the_reference_domain():
    # wherever the reference plans a shape (tc/params.py:225-267 with its
    # 63-bit table) and the product fits a B200's 180 GB, plan_gpu plans it
    rng = random.Random(5)
    shapes = [((1 << 22) + 1, 64), (1 << 23, 64), (1 << 24, 64), ((1 << 24) + 1, 64), (1 << 25, 64),
              (1 << 26, 64), (16, (1 << 21) + 1), (2, (1 << 22) + 1), (1, 1 << 24), (16, 300000),
              (2, 500000), (1 << 22, 1024), (1 << 20, 4096), (4096, 1 << 17), (1, 2), (3, 1)]
    shapes += [(rng.randint(1, 1 << rng.randint(1, 26)), rng.randint(1, 1 << rng.randint(1, 22)))
               for _ in range(120)]
    checked = 0
    for d, n_in in shapes:
        dmin = rng.choice([d, max(1, d // 3), 1])
        try:
            params.plan_from_shape(d, n_in, 2)
        except Exception:                       # the reference does not plan it either
            continue
        cw = -(-n_in // 64)
        out_cw = -(-params.product_width_bits(d, n_in) // 64)
        if (d + dmin) * cw * 8 + (d + dmin - 1) * out_cw * 8 > 60e9 or 2.5 * (d + dmin) * n_in > 180e9:
            continue                            # operands + product, or the grids (~17x the
                                                # operands' bytes), beyond one device
        pl = params.plan_gpu(d, dmin, n_in)
        need = params.plan_device_bytes(pl, d, dmin)
        if need > 180e9:
            continue                            # beyond one device; DeviceError names the size
        _check_plan(pl, d, dmin, n_in)
        checked += 1
    assert checked > 60


def test_split_plans_for_the_verdict_shapes():
    for d, n_in, kind in (((1 << 22) + 1, 64, None), (1 << 23, 64, None), (1 << 25, 64, SPLIT_POLY),
                          (16, (1 << 21) + 1, SPLIT_COEF), (2, (1 << 22) + 1, SPLIT_COEF),
                          (2, 500000, SPLIT_COEF)):
        pl = params.plan_gpu(d, d, n_in)
        assert (pl.split.kind if pl.split else None) == kind, pl.describe()
        _check_plan(pl, d, d, n_in)
    # the ADVICE case: a direct plan whose final tiles would not fit is never chosen
    pl = params.plan_gpu(16, 16, 300000)
    assert params.final_tile_bytes(pl.K, pl.s_y, pl.P) <= params.FINAL_SMEM_LIMIT


def test_forced_splits_plan():
    pl = params.plan_with_split(10, 7, 500, SplitSpec(SPLIT_COEF, 4, 128, 16))
    assert pl.split.n == 4 and pl.d == 10 + 3 * 16
    pl = params.plan_with_split(100, 100, 50, SplitSpec(SPLIT_POLY, 7, 128, 16))
    assert pl.d == 16 and pl.n_in == 6 * 128 + 51
    with pytest.raises(ValueError):
        params.plan_with_split(10, 7, 500, SplitSpec(SPLIT_COEF, 4, 128, 15))
