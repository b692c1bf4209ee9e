"""GPU parity: the CUDA path (through libtcgpu.so's C-ABI) against the golden
vectors produced by the reference and against the CPU oracle.  Integer work:
every comparison is bit-exact (zero tolerance)."""
import json
import os
import random

import numpy as np
import pytest

from conftest import GOLDEN, load_golden

pytestmark = pytest.mark.gpu

import paper_1612_05778_b200 as tc  # noqa: E402
from paper_1612_05778_b200 import seams, workloads  # noqa: E402
from paper_1612_05778_b200.params import gpu_prime_table, plan_gpu  # noqa: E402


def _poly(words, bits):
    return tc.IntPolynomial(np.ascontiguousarray(words), bits)


def _random_poly(rng, d, nbits, extremes=False):
    lo, hi = -(1 << (nbits - 1)), (1 << (nbits - 1)) - 1
    while True:
        if extremes:
            coeffs = [rng.choice([lo, hi]) for _ in range(d)]
        else:
            coeffs = [rng.randint(lo, hi) for _ in range(d)]
            if rng.random() < 0.4:
                coeffs[rng.randrange(d)] = lo
            if rng.random() < 0.4:
                coeffs[rng.randrange(d)] = hi
        if any(coeffs):
            return tc.IntPolynomial.from_coefficients(coeffs, bit_width=nbits)


# ---------------------------------------------------------------- field / NTT

def test_modmul_probe_matches_bigint():
    rng = np.random.default_rng(99)
    for spec in gpu_prime_table()[:4]:
        p = spec.p
        a = rng.integers(0, p, size=5000, dtype=np.uint64).astype(np.uint32)
        b = rng.integers(0, p, size=5000, dtype=np.uint64).astype(np.uint32)
        got = seams.modmul(p, a, b, mode=0)
        exp = (a.astype(object) * b.astype(object)) % p
        assert np.array_equal(got.astype(object), exp)
        got = seams.modmul(p, a, b, mode=1)
        rinv = pow(1 << 32, -1, p)
        exp = (a.astype(object) * b.astype(object) * rinv) % p
        assert np.array_equal(got.astype(object), exp)


def test_ntt_probe_delta_inverse_linearity():
    # pkg/tests/test_ntt2d.py:36-81 restated for the device transform
    rng = random.Random(17)
    spec = gpu_prime_table()[0]
    p, g = spec.p, spec.generator
    for logn in range(1, 14):
        n = 1 << logn
        delta = np.zeros(n, dtype=np.uint32)
        delta[0] = 1
        assert np.all(seams.ntt(delta, p, g) == 1)
        v = np.array([rng.randrange(p) for _ in range(n)], dtype=np.uint32)
        assert np.array_equal(seams.ntt(seams.ntt(v, p, g), p, g, inverse=True), v)
    n = 64
    u = np.array([rng.randrange(p) for _ in range(n)], dtype=np.uint64)
    w = np.array([rng.randrange(p) for _ in range(n)], dtype=np.uint64)
    al, be = rng.randrange(p), rng.randrange(p)
    mix = ((al * u.astype(object) + be * w.astype(object)) % p).astype(np.uint32)
    fu, fw, fm = (seams.ntt(x.astype(np.uint32), p, g).astype(object) for x in (u, w, mix))
    assert all((al * x + be * y) % p == z for x, y, z in zip(fu, fw, fm))


# ---------------------------------------------------------------- ConvertIn

def test_digits_match_reference_golden():
    meta, arr = load_golden("digits")
    for m in meta:
        words = arr[f"d{m['id']}_in"]
        poly = _poly(words, m["bits"])
        if m["error"]:
            with pytest.raises(tc.EncodingError):
                seams.digits(poly, m["K"], m["M"])
            continue
        got = seams.digits(poly, m["K"], m["M"])
        assert np.array_equal(got, arr[f"d{m['id']}_digits"]), m


def test_digits_match_oracle_wide_rows(oracle):
    # long carry chains across warps and rounds: K up to 8192, all-ones rows
    rng = np.random.default_rng(3)
    for K, M, d in ((8192, 33, 3), (2048, 33, 5), (64, 63, 40), (1, 40, 70), (4096, 17, 2)):
        N = K * M
        nl = -(-N // 64)
        words = rng.integers(0, 2**64 - 1, endpoint=True, size=(d, nl), dtype=np.uint64)
        words[0, :] = np.uint64(0xFFFFFFFFFFFFFFFF)
        if d > 2:
            words[2, :] = 0
        # clear bits >= N-2 so every row is within capacity, keep sign extension
        top = (N - 2)
        for i in range(d):
            v = int.from_bytes(words[i].tobytes(), "little") & ((1 << top) - 1)
            if i % 2:
                v -= 1 << (top - 1)
            words[i] = np.frombuffer((v & ((1 << (64 * nl)) - 1)).to_bytes(8 * nl, "little"), dtype=np.uint64)
        plan = oracle.MulPlan(d=d, N=N, K=K, M=M, s_y=1, primes=(), e=0, f=0)
        exp = oracle.digits(words, N, plan)
        got = seams.digits(_poly(words, N), K, M)
        assert np.array_equal(got, exp), (K, M)


# ---------------------------------------------------------------- convolutions / CRT

def test_c_plus_minus_match_reference_golden():
    meta, arr = load_golden("cpm")
    ran = 0
    for m in meta:
        n, d, K, M = m["id"], m["d"], m["K"], m["M"]
        da, db = arr[f"m{n}_a"], arr[f"m{n}_b"]
        N = K * M
        vals = [[sum(int(x) << (M * j) for j, x in enumerate(row)) for row in dg] for dg in (da, db)]
        if any(not -(1 << (N - 1)) <= v < (1 << (N - 1)) for vs in vals for v in vs):
            continue   # balanced capacity exceeds the N-bit range: not an N-bit input
        a, b = (tc.IntPolynomial.from_coefficients(vs, bit_width=N) for vs in vals)
        if a.is_zero() or b.is_zero():
            continue
        ran += 1
        plan = plan_gpu(d, d, N, K=K, M=M)
        full, _ = seams.bivariate_product(a, b, plan)
        cp, cm = seams.fold_c_plus_minus(full, K)
        e = m["plan"]["e"]
        assert np.array_equal(seams.ints_to_limbs(cp, e), arr[f"m{n}_cp"]), m
        assert np.array_equal(seams.ints_to_limbs(cm, e), arr[f"m{n}_cm"]), m
    assert ran >= len(meta) // 3


@pytest.mark.parametrize("mlo,mhi,seed", [(2, 40, 31), (41, 63, 32)])
def test_bivariate_product_vs_naive(oracle, mlo, mhi, seed):
    # exact c_ij (k_final's DUMP mode) for P = 1..5 primes
    rng = random.Random(seed)
    for _ in range(20):
        d = rng.randint(1, 9)
        K = rng.choice([1, 2, 4, 8])
        M = rng.randint(mlo, mhi)
        half = 1 << (M - 1)
        dg = lambda: np.array([[rng.randint(-half, half - 1) for _ in range(K)] for _ in range(d)],
                              dtype=np.int64)
        A, B = dg(), dg()
        N = K * M
        vals = [[sum(int(v) << (M * j) for j, v in enumerate(row)) for row in x] for x in (A, B)]
        if any(not -(1 << (N - 1)) <= v < (1 << (N - 1)) for vs in vals for v in vs):
            continue
        a, b = (tc.IntPolynomial.from_coefficients(vs, bit_width=N) for vs in vals)
        if a.is_zero() or b.is_zero():
            continue
        full, plan = seams.bivariate_product(a, b, plan_gpu(d, d, K * M, K=K, M=M))
        exp = oracle.naive_bivariate(A, B, K)
        assert [row[:2 * K - 1] for row in full] == exp
        assert all(row[2 * K - 1] == 0 for row in full)


# ---------------------------------------------------------------- products

def test_products_match_reference_golden():
    meta, arr = load_golden("products")
    for m in meta:
        a = _poly(arr[f"c{m['id']}_a"], m["a_bits"])
        b = _poly(arr[f"c{m['id']}_b"], m["b_bits"])
        out = tc.multiply(tc.MulRequest(a, b, prime_count=m["prime_count"]))
        assert out.bit_width == m["out_bits"]
        assert np.array_equal(out.words, arr[f"c{m['id']}_out"]), m


def test_products_match_oracle_random(oracle):
    rng = random.Random(8080)
    for _ in range(40):
        a = _random_poly(rng, rng.randint(1, 300), rng.randint(1, 700))
        b = _random_poly(rng, rng.randint(1, 300), rng.randint(1, 700))
        out = tc.multiply(tc.MulRequest(a, b))
        exp, bits = oracle.multiply_words(a.words, a.bit_width, b.words, b.bit_width)
        assert out.bit_width == bits and np.array_equal(out.words, exp)


def test_known_answers():
    one = tc.IntPolynomial.from_coefficients([1])
    assert tc.multiply(tc.MulRequest(one, one)).coefficients() == [1]
    out = tc.multiply(tc.MulRequest(tc.IntPolynomial.from_coefficients([1, 1]),
                                    tc.IntPolynomial.from_coefficients([-1, 1])))
    assert out.coefficients() == [-1, 0, 1]
    x = 3 ** 400
    a = tc.IntPolynomial.from_coefficients([x])
    b = tc.IntPolynomial.from_coefficients([-(5 ** 340)])
    assert tc.multiply(tc.MulRequest(a, b)).coefficients() == [-x * 5 ** 340]
    a = tc.IntPolynomial.from_coefficients([1, -2, 3])
    b = tc.IntPolynomial.from_coefficients([5, 7])
    assert tc.multiply(tc.MulRequest(a, b)).coefficients() == [5, -3, 1, 21]


def test_extremes_mixed_widths_and_invariance(oracle):
    rng = random.Random(7)
    for d, nbits in ((1, 8), (5, 16), (17, 64), (33, 1025), (3, 4097)):
        a = _random_poly(rng, d, nbits, extremes=True)
        out = tc.multiply(tc.MulRequest(a, a))
        exp, bits = oracle.multiply_words(a.words, a.bit_width, a.words, a.bit_width)
        assert np.array_equal(out.words, exp)
    a = _random_poly(rng, 9, 300)
    b = _random_poly(rng, 4, 3)
    for x, y in ((a, b), (b, a)):
        exp, _ = oracle.multiply_words(x.words, x.bit_width, y.words, y.bit_width)
        assert np.array_equal(tc.multiply(tc.MulRequest(x, y)).words, exp)
    a = _random_poly(rng, 40, 120)
    b = _random_poly(rng, 37, 120)
    base = tc.multiply(tc.MulRequest(a, b))
    for pc in (1, 2, 3):
        for w in (None, 1, 2, 8):
            assert tc.multiply(tc.MulRequest(a, b, prime_count=pc, worker_hint=w)) == base


def test_explicit_plans_agree():
    rng = random.Random(21)
    a = _random_poly(rng, 200, 500)
    b = _random_poly(rng, 150, 500)
    base = tc.multiply(tc.MulRequest(a, b))
    for K in (8, 16, 32, 128, 512):
        out, _, plan = tc.multiply_with_plan(tc.MulRequest(a, b), K=K)
        assert out == base, plan.describe()


def test_errors():
    zero = tc.IntPolynomial.from_coefficients([0, 0])
    with pytest.raises(tc.EmptyInputError):
        tc.multiply(tc.MulRequest(zero, tc.IntPolynomial.from_coefficients([1])))
    a = tc.IntPolynomial.from_coefficients([1, 2])
    with pytest.raises(ValueError):
        tc.multiply(tc.MulRequest(a, a, prime_count=4))
    # prime_count=1 plans like the reference (which recovers this with one
    # 63-bit prime at M=16) and never changes the product
    big = tc.IntPolynomial.from_coefficients([(1 << 1999) - 1] * 64)
    assert tc.multiply(tc.MulRequest(big, big, prime_count=1)) == tc.multiply(tc.MulRequest(big, big))


def test_stats_accounting():
    rng = random.Random(41)
    a = _random_poly(rng, 256, 256)
    b = _random_poly(rng, 256, 256)
    poly, stats = tc.multiply_with_stats(tc.MulRequest(a, b, worker_hint=2))
    assert stats.workers == 2
    assert poly == tc.multiply(tc.MulRequest(a, b))
    assert stats.total > 0 and stats.stage_sum() <= stats.total
    # the reference's stage meaning (tc/multiplier.py:131-166): every stage of
    # the fused kernels is attributed, transfers reported apart
    for name in ("convert", "ntt_forward", "pointwise", "ntt_inverse", "crt", "recover", "h2d", "d2h"):
        assert getattr(stats, name) > 0, (name, stats)
    assert stats.stage_sum() + stats.h2d + stats.d2h <= stats.total
    for name in ("C2", "C5"):            # the other k_final paths (warp-group ConvertOut), sizeable stages
        (aw, ab), (bw, bb) = workloads.make_inputs(name)
        p, st = tc.multiply_with_stats(tc.MulRequest(tc.IntPolynomial._trusted(aw, ab), tc.IntPolynomial._trusted(bw, bb)))
        assert st.crt > 0 and st.recover > 0 and st.pointwise > 0 and st.convert > 0, st
        assert p == tc.multiply(tc.MulRequest(tc.IntPolynomial._trusted(aw, ab), tc.IntPolynomial._trusted(bw, bb)))


# ---------------------------------------------------------------- full BASELINE sizes

@pytest.mark.parametrize("name", ["C1", "C2", "C4", "C5", "C3"])
def test_full_config_matches_reference_hash(name, oracle):
    cfg = json.load(open(os.path.join(GOLDEN, "configs.json")))[name]
    (aw, ab), (bw, bb) = workloads.make_inputs(name)
    assert workloads.words_sha256(aw) == cfg["a_sha256"]
    a, b = tc.IntPolynomial._trusted(aw, ab), tc.IntPolynomial._trusted(bw, bb)
    out = tc.multiply(tc.MulRequest(a, b))
    assert out.bit_width == cfg["out_bits"] and list(out.words.shape) == cfg["out_shape"]
    assert workloads.words_sha256(out.words) == cfg["out_sha256"]
    # size-independent property: c(r) == a(r) b(r) mod q
    q, r = (1 << 61) - 1, 0x1234567890ABCDE
    assert oracle.eval_mod(out.words, q, r) == oracle.eval_mod(aw, q, r) * oracle.eval_mod(bw, q, r) % q


# ---------------------------------------------------------------- sharded (multi-GPU) path

@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("mode", ["rows", "primes"])
def test_sharded_product_virtual_ranks(world, mode, oracle):
    # the multi-GPU decompositions run as `world` virtual ranks (contexts,
    # threads, copy-stream exchanges) on one GPU: the row split (compact
    # inputs, two transposes) and the prime split (world <= P)
    from paper_1612_05778_b200 import shard
    rng = random.Random(world * 7 + len(mode))
    for d, nbits in ((300, 500), (1000, 2000), (64, 4097), (5, 63)):
        a = _random_poly(rng, d, nbits)
        b = _random_poly(rng, max(1, d - 7), nbits)
        plan = plan_gpu(d, max(1, d - 7), nbits)
        if mode == "primes" and world > plan.P:
            continue
        try:
            out, plan = shard.multiply_local(a, b, world, mode=mode)
        except tc.DeviceError as ex:              # a grid too small to split this many ways
            assert "does not split" in str(ex) or "too small" in str(ex), ex
            continue
        assert out == tc.multiply(tc.MulRequest(a, b)), plan.describe()


@pytest.mark.parametrize("name,world,mode", [("C1", 4, "rows"), ("C2", 4, "rows"), ("C5", 4, "rows"),
                                             ("C2", 4, "primes"), ("C4", 4, "rows"), ("C4", 4, "primes"),
                                             ("C3", 2, "primes"), ("C3", 2, "rows"), ("C3", 8, "rows")])
def test_sharded_full_config(name, world, mode):
    from paper_1612_05778_b200 import shard
    cfg = json.load(open(os.path.join(GOLDEN, "configs.json")))[name]
    (aw, ab), (bw, bb) = workloads.make_inputs(name)
    a, b = tc.IntPolynomial._trusted(aw, ab), tc.IntPolynomial._trusted(bw, bb)
    out, plan = shard.multiply_local(a, b, world, mode=mode)
    assert out.bit_width == cfg["out_bits"]
    assert workloads.words_sha256(out.words) == cfg["out_sha256"], (name, world, mode, plan.describe())


def test_worker_hint_uses_the_gpus_present():
    # worker_hint maps to the GPU count; never changes the product
    from paper_1612_05778_b200 import multiplier, shard
    n = shard.device_count()
    assert multiplier._gpus_for(None) == 1 and multiplier._gpus_for(1) == 1
    assert multiplier._gpus_for(64) == 1 << (n.bit_length() - 1)
    rng = random.Random(3)
    a, b = _random_poly(rng, 200, 700), _random_poly(rng, 150, 700)
    base = tc.multiply(tc.MulRequest(a, b))
    p, st = tc.multiply_with_stats(tc.MulRequest(a, b, worker_hint=8))
    assert p == base and st.workers == 8 and st.gpus == multiplier._gpus_for(8)


def _dist_worker(rank, world, port, name, mode, result):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1612_05778_b200 import shard
    (aw, ab), (bw, bb) = workloads.make_inputs(name)
    a, b = tc.IntPolynomial._trusted(aw, ab), tc.IntPolynomial._trusted(bw, bb)
    dm = shard.DistributedMultiplier(0, mode=mode)
    out, plan = dm.multiply(a, b)
    local, _ = dm.multiply(a, b, to_host="local")     # this rank's rows, strided into a full-size buffer
    if mode == "primes":
        dm.upload(a, b)
        out2, _ = dm.multiply(a, b, resident=True)
    else:
        out2 = out
    lw = (world - 1).bit_length()
    c0 = int(format(rank, f"0{lw}b")[::-1], 2) if lw else 0
    result[f"rows{rank}"] = workloads.words_sha256(np.ascontiguousarray(local[c0::world]))
    if rank == 0:
        result["sha"] = workloads.words_sha256(out.words)
        result["sha2"] = workloads.words_sha256(out2.words)
        for r in range(world):
            c = int(format(r, f"0{lw}b")[::-1], 2) if lw else 0
            result[f"exp{r}"] = workloads.words_sha256(np.ascontiguousarray(out.words[c::world]))
    dist.destroy_process_group()


@pytest.mark.parametrize("name,mode", [("C1", "rows"), ("C2", "rows"), ("C2", "primes")])
def test_distributed_multiplier_two_processes(name, mode):
    # the real multi-process code path (DistributedMultiplier, torch.distributed
    # exchanges) with 2 ranks sharing this one GPU; gloo stages the exchanges
    # through host memory, so no kernel waits on another process
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    result = mp.Manager().dict()
    mp.spawn(_dist_worker, args=(2, port, name, mode, result), nprocs=2, join=True)
    cfg = json.load(open(os.path.join(GOLDEN, "configs.json")))[name]
    assert result["sha"] == cfg["out_sha256"] and result["sha2"] == cfg["out_sha256"]
    for r in range(2):      # each rank's direct download holds exactly its rows of the product
        assert result[f"rows{r}"] == result[f"exp{r}"]


def test_corruption_is_detected():
    # tc/multiplier.py:59-63: a residue that fails the CRT bound check raises
    # CorruptedConvolutionError naming the slot; injected through plan.flags
    from paper_1612_05778_b200.multiplier import _run_pipeline
    rng = random.Random(77)
    a = _random_poly(rng, 40, 300)
    b = _random_poly(rng, 40, 300)
    for row in (0, 5, 78):
        with pytest.raises(tc.CorruptedConvolutionError, match=rf"\({row}, 1\)"):
            _run_pipeline(tc.MulRequest(a, b), plan_override={"flags": 1 | (row << 16)})
    assert tc.multiply(tc.MulRequest(a, b)) == tc.multiply(tc.MulRequest(b, a))   # no fault: fine


def test_odd_combination_is_detected():
    # tc/_kernels.py:416-417 -> tc/multiplier.py:156-160: the reference's u + v
    # parity check; here the acyclic product's term 2K-1 of a row must be 0.
    # plan.flags bit 1 adds 1 to every residue of slot (row, 2K-1): a value
    # inside the CRT bound, so only this check can catch it
    from paper_1612_05778_b200.multiplier import _run_pipeline
    rng = random.Random(78)
    a = _random_poly(rng, 40, 300)
    b = _random_poly(rng, 33, 300)
    for row in (0, 7, 71):
        with pytest.raises(tc.CorruptedConvolutionError, match=rf"odd combination at coefficient {row}$"):
            _run_pipeline(tc.MulRequest(a, b), plan_override={"flags": 2 | (row << 16)})
    # a padding row past the product is never checked
    out, _, _ = _run_pipeline(tc.MulRequest(a, b), plan_override={"flags": 2 | (200 << 16)})
    assert out == tc.multiply(tc.MulRequest(a, b))


def test_extreme_plans(oracle):
    # K = 1 (no digit split), one prime, and the widest prime sets the planner
    # reaches with single-word digits; every plan gives the same product
    rng = random.Random(99)
    cases = [(5, 12, dict(K=1)), (4, 8, {}), (64, 60, dict(K=1)), (300, 63, dict(K=1)),
             (2048, 63, dict(K=1)), (2048, 126, dict(K=4)), (33, 1000, dict(K=16))]
    for d, nbits, kw in cases:
        a = _random_poly(rng, d, nbits)
        b = _random_poly(rng, d, nbits)
        out, _, plan = tc.multiply_with_plan(tc.MulRequest(a, b), **kw)
        exp, bits = oracle.multiply_words(a.words, a.bit_width, b.words, b.bit_width)
        assert out.bit_width == bits and np.array_equal(out.words, exp), plan.describe()
    p1 = plan_gpu(4, 4, 8)
    assert p1.P == 1
    wide = plan_gpu(2048, 2048, 63, K=1)
    assert wide.P >= 5
    # an explicit split too narrow for the operands is the reference's EncodingError
    a = _random_poly(rng, 8, 126, extremes=True)
    with pytest.raises(tc.EncodingError):
        tc.multiply_with_plan(tc.MulRequest(a, a), K=2, M=63)


def test_two_word_digits(oracle):
    # 64 <= M <= 126: digits of two words (planner's choice for C1/C2/C3/C5
    # widths); random, extreme (most negative, all-ones) and mixed-width
    # operands against the oracle, and the digit-capacity EncodingError
    rng = random.Random(6565)
    cases = [(40, 33, 129, dict(K=2, M=65)), (300, 300, 1025, dict(K=16, M=65)), (128, 100, 4000, dict(K=64, M=64)),
             (64, 64, 2000, dict(K=16, M=126)), (500, 20, 700, dict(K=8, M=90)), (7, 9, 8193, dict(K=128, M=65)),
             (256, 256, 1025, dict(K=16, M=65)), (3, 2, 126, dict(K=1, M=126)), (1000, 1000, 65, dict(K=1, M=65))]
    for da, db, nbits, kw in cases:
        for extremes in (False, True):
            a = _random_poly(rng, da, nbits, extremes=extremes)
            b = _random_poly(rng, db, max(2, nbits - rng.randrange(0, 60)), extremes=extremes)
            out, _, plan = tc.multiply_with_plan(tc.MulRequest(a, b), **kw)
            assert plan.M > 63, plan.describe()
            exp, bits = oracle.multiply_words(a.words, a.bit_width, b.words, b.bit_width)
            assert out.bit_width == bits and np.array_equal(out.words, exp), (da, db, nbits, plan.describe())
    a = _random_poly(rng, 8, 300, extremes=True)
    with pytest.raises(tc.EncodingError):
        tc.multiply_with_plan(tc.MulRequest(a, a), K=2, M=100)


def test_block_convert_out_carry_chains(oracle):
    # M = 65 with rows of >= 64 terms (crt_convert_block64: 64-term blocks, 64-bit digits, segments
    # fixed up after a barrier): operands whose products carry across every block and segment boundary
    # (all-ones and sign-alternating coefficients), few rows (many segments per row) and many, P = 3..6
    rng = random.Random(6564)
    def const_poly(d, nbits, pattern):
        limbs = -(-nbits // 64)
        w = np.zeros((d, limbs), dtype=np.uint64)
        for i in range(d):
            v = pattern(i)
            v &= (1 << (64 * limbs)) - 1
            for k in range(limbs):
                w[i, k] = (v >> (64 * k)) & 0xFFFFFFFFFFFFFFFF
        return _poly(w, nbits)
    cases = [(1, 1, 2070, 32), (2, 1, 4150, 64), (3, 3, 4100, 64), (1, 2, 66000, 1024), (5, 4, 33000, 512),
             (40, 33, 8300, 128), (300, 7, 2070, 32), (1, 1, 16600, 256)]
    for da, db, nbits, K in cases:
        top = (1 << (nbits - 1)) - 1
        pats = [(lambda i: top, lambda i: top), (lambda i: -top, lambda i: top),
                (lambda i: top if i % 2 else -top, lambda i: -top - 1 + (i % 3)),
                (lambda i: (1 << (nbits - 2)) + i, lambda i: -1 - i)]
        for pa, pb in pats:
            a, b = const_poly(da, nbits, pa), const_poly(db, nbits, pb)
            out, _, plan = tc.multiply_with_plan(tc.MulRequest(a, b), K=K, M=65)
            assert plan.M == 65 and plan.K == K, plan.describe()
            exp, bits = oracle.multiply_words(a.words, a.bit_width, b.words, b.bit_width)
            assert out.bit_width == bits and np.array_equal(out.words, exp), (da, db, nbits, plan.describe())
        a = _random_poly(rng, da, nbits, extremes=True)
        b = _random_poly(rng, db, nbits, extremes=True)
        out, _, plan = tc.multiply_with_plan(tc.MulRequest(a, b), K=K, M=65)
        exp, bits = oracle.multiply_words(a.words, a.bit_width, b.words, b.bit_width)
        assert out.bit_width == bits and np.array_equal(out.words, exp), (da, db, nbits, plan.describe())


def test_chunked_upload_unbalanced(oracle):
    # multiply() uploads large operands in chunks and starts the first pass of the CTAs that read a
    # chunk as it lands (k_low in bit-reversed CTA order): unbalanced lengths, so chunks clip at d
    # and whole chunks of the shorter operand are empty; pageable and page-locked sources
    from paper_1612_05778_b200 import _lib
    rng = np.random.default_rng(20000)
    def rand_words(d, nbits):
        limbs = -(-nbits // 64)
        w = rng.integers(0, 2**64 - 1, endpoint=True, size=(d, limbs), dtype=np.uint64)
        top = nbits - 64 * (limbs - 1)                      # sign-extend bit nbits-1 through the top limb
        if top < 64:
            sign = (w[:, -1] >> np.uint64(top - 1)) & np.uint64(1)
            keep = (np.uint64(1) << np.uint64(top)) - np.uint64(1)
            w[:, -1] = (w[:, -1] & keep) | np.where(sign == 1, ~keep, np.uint64(0))
        return w
    for da, db, nbits in [(20000, 3000, 16384), (2500, 18000, 20001)]:
        aw, bw = rand_words(da, nbits), rand_words(db, nbits)
        exp, bits = oracle.multiply_words(aw, nbits, bw, nbits)
        out = tc.multiply(tc.MulRequest(_poly(aw, nbits), _poly(bw, nbits)))
        assert out.bit_width == bits and np.array_equal(out.words, exp), (da, db, nbits)
        pa = _lib.pinned.empty(aw.shape, np.uint64); pa[...] = aw
        pb = _lib.pinned.empty(bw.shape, np.uint64); pb[...] = bw
        out = tc.multiply(tc.MulRequest(tc.IntPolynomial._trusted(pa, nbits), tc.IntPolynomial._trusted(pb, nbits)))
        assert out.bit_width == bits and np.array_equal(out.words, exp), (da, db, nbits, "pinned")


def test_plan_sweep(oracle):
    # every transform length 2K = 2 .. 2^14 (the compile-time x schedules, the
    # fused twist / duplication rounds, k_high_ct / generic passes), degrees
    # that move the in-tile y levels yl across their range, unbalanced
    # operands and explicit digit sizes: bit-exact against the oracle
    rng = random.Random(2024)
    cases = []
    for lgk in range(0, 14):
        K = 1 << lgk
        for d, nbits, db in ((3, 20, 3), (40, 60, 17), (700, 50, 700)):
            nb = max(2, min(K * 31, nbits * (1 + lgk)))       # widths that want about this K
            if d * nb > 3_000_000:
                continue
            cases.append((d, db, nb, dict(K=K)))
    cases += [(1, 1, 5, {}), (2, 1, 63, {}), (1, 300, 64, {}), (2047, 3, 33, {}), (5000, 5000, 31, {}),
              (1000, 1000, 200, dict(M=25)), (64, 64, 4000, dict(M=40)), (257, 255, 129, dict(M=63))]
    for da, db, nbits, kw in cases:
        a = _random_poly(rng, da, nbits)
        b = _random_poly(rng, db, nbits)
        try:
            out, _, plan = tc.multiply_with_plan(tc.MulRequest(a, b), **kw)
        except tc.EncodingError:
            continue                     # an explicit split too narrow for the operands
        exp, bits = oracle.multiply_words(a.words, a.bit_width, b.words, b.bit_width)
        assert out.bit_width == bits and np.array_equal(out.words, exp), (da, db, nbits, plan.describe())
