"""Randomised GPU-vs-oracle sweep over shapes and explicit plans (not part of the test suite:
a longer soak of the k_low / k_final code paths).  usage: python tools/stress.py [seconds] [seed]"""
import sys, time, random
import numpy as np
sys.path.insert(0, '.')
import paper_1612_05778_b200 as tc
from oracle import port

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
LARGE = len(sys.argv) > 3 and sys.argv[3] == "large"
nrng = np.random.default_rng(rng.randrange(1 << 30))


def rand_words(d, nbits, mode):
    limbs = -(-nbits // 64)
    if mode == 0:
        w = nrng.integers(0, 2**64 - 1, endpoint=True, size=(d, limbs), dtype=np.uint64)
    elif mode == 1:                                   # all-ones magnitudes / most negative
        w = np.full((d, limbs), 0xFFFFFFFFFFFFFFFF, dtype=np.uint64)
        w[nrng.random(d) < 0.5] = 0
    else:                                             # sparse
        w = np.zeros((d, limbs), dtype=np.uint64)
        idx = nrng.integers(0, d, size=max(1, d // 7))
        w[idx] = nrng.integers(0, 2**64 - 1, endpoint=True, size=(len(idx), limbs), dtype=np.uint64)
    top = nbits - 64 * (limbs - 1)
    if top < 64:
        sign = (w[:, -1] >> np.uint64(top - 1)) & np.uint64(1)
        keep = (np.uint64(1) << np.uint64(top)) - np.uint64(1)
        w[:, -1] = (w[:, -1] & keep) | np.where(sign == 1, ~keep, np.uint64(0))
    if not w.any():
        w[0, 0] = 1
    return w


t0, n, by_plan = time.time(), 0, {}
while time.time() - t0 < budget:
    kind = rng.random()
    if LARGE and rng.random() < 0.5:   # tens of MB per operand: chunked uploads, several k_final chunks
        da, nbits = rng.choice([(60000, 4000), (3000, 70000), (200000, 700), (12000, 20000), (40, 900000), (500000, 130)])
        db = max(1, int(da * rng.choice([1.0, 0.5, 0.03])))
        kw = {}
    elif kind < 0.45:        # M = 65 plans with rows of >= 64 terms (block ConvertOut), few to many rows
        K = rng.choice([32, 64, 128, 256, 512, 1024, 2048])
        nbits = rng.randrange(65 * K - 120, 65 * K - 2)
        da, db = rng.choice([(1, 1), (2, 3), (5, 1), (17, 40), (130, 7), (300, 300), (1000, 2)])
        kw = dict(K=K, M=65)
    elif kind < 0.7:       # planner's choice, mixed sizes
        da, db = rng.randrange(1, 3000), rng.randrange(1, 3000)
        nbits = rng.randrange(2, 9000)
        kw = {}
    elif kind < 0.85:      # single-word digits
        K = rng.choice([1, 2, 8, 32, 128])
        M = rng.choice([20, 33, 50, 63])
        nbits = max(2, K * M - rng.randrange(1, 40))
        da, db = rng.randrange(1, 2000), rng.randrange(1, 2000)
        kw = dict(K=K, M=M)
    else:                  # other two-word digit widths
        K = rng.choice([4, 16, 64, 256])
        M = rng.choice([64, 66, 80, 96, 97, 126])
        nbits = max(2, K * M - rng.randrange(2, 60))
        da, db = rng.randrange(1, 600), rng.randrange(1, 600)
        kw = dict(K=K, M=M)
    mode = rng.randrange(3)
    aw, bw = rand_words(da, nbits, mode), rand_words(db, nbits, rng.randrange(3))
    a, b = tc.IntPolynomial(aw, nbits), tc.IntPolynomial(bw, nbits)
    try:
        out, _, plan = tc.multiply_with_plan(tc.MulRequest(a, b), **kw)
    except (tc.PrimeCapacityError, tc.EncodingError, ValueError) as ex:
        continue
    exp, bits = port.multiply_words(aw, nbits, bw, nbits)
    ok = out.bit_width == bits and np.array_equal(out.words, exp)
    key = (plan.K, plan.M, plan.P)
    by_plan[key] = by_plan.get(key, 0) + 1
    n += 1
    if not ok:
        print("MISMATCH", da, db, nbits, kw, plan.describe(), flush=True)
        sys.exit(1)
print(f"{n} products ok in {time.time() - t0:.0f} s; plans (K, M, P): {sorted(by_plan.items())[:60]}")
