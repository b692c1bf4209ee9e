# Emulate k_final's ConvertOut (rounds of 512 threads, warps of 32) on exact terms
import random
def conv_out_emu(terms, M, P, W32, blockDim=512):
    # terms: list of rows, each list of L ints (exact c_ij); returns list of rows of W32 u32 words
    R = len(terms); L = len(terms[0])
    def limbs(v):
        v &= (1 << (32*P)) - 1
        return [(v >> (32*l)) & 0xffffffff for l in range(P)]
    T = [[limbs(v) for v in row] for row in terms]
    total = R * W32
    out = [[0]*W32 for _ in range(R)]
    s_carry, s_hi = 0, 0
    def tf_of(x):
        return tuple(((x + c) >> 32) for c in (-1, 0, 1))
    ident = (-1, 0, 1)
    def comp(g, f):  # g o f
        return tuple(g[v+1] for v in f)
    for gb in range(0, total, blockDim):
        xs, fs, his, rws = [], [], [], []
        for t in range(blockDim):
            gi = gb + t
            valid = gi < total
            r = gi // W32 if valid else R
            w = gi - r*W32 if valid else 0
            s = 0
            if valid:
                lo_n = 32*(w-P)
                jf = 0 if lo_n <= 0 else (lo_n + M - 1)//M
                jl = min(L-2, (32*w+31)//M)
                for j in range(jf, jl+1):
                    bit = M*j; k = w - (bit >> 5); rr = bit & 31
                    c = T[r][j]
                    sgn = 0xffffffff if c[P-1] >> 31 else 0
                    cur = c[k] if k < P else sgn
                    prv = c[k-1] if k > 0 else 0
                    piece = ((cur << rr) | (prv >> (32-rr))) & 0xffffffff if rr else cur
                    if k < P: s += piece
                    else: s += piece - (1 << 32) if piece >> 31 else piece
            his.append(s >> 32); xs.append((valid, r, w, s))
        res = []
        for t in range(blockDim):
            valid, r, w, s = xs[t]
            hprev = his[t-1] if t > 0 else s_hi
            x = (s & 0xffffffff) + (0 if w == 0 else hprev)
            if not valid: f = ident
            elif w == 0: c0 = tf_of(x)[1]; f = (c0, c0, c0)
            else: f = tf_of(x)
            fs.append(f); res.append(x)
        # sequential exclusive prefix
        c = s_carry
        for t in range(blockDim):
            valid, r, w, s = xs[t]
            if valid:
                out[r][w] = (res[t] + (0 if w == 0 else c)) & 0xffffffff
            c = fs[t][c+1]
        s_carry = c; s_hi = his[-1]
    return out

def check(R, K, M, P, dmul):
    L = 2*K
    bound = dmul * K << (2*M-2)
    terms = [[random.randint(-bound, bound) for _ in range(L-1)] + [0] for _ in range(R)]
    vals = [sum(v << (M*j) for j, v in enumerate(row)) for row in terms]
    nb = max(abs(v) for v in vals).bit_length() + 2
    W32 = 2 * ((nb + 63)//64)
    out = conv_out_emu(terms, M, P, W32)
    for r in range(R):
        u = sum(wd << (32*i) for i, wd in enumerate(out[r]))
        if u >> (32*W32 - 1): u -= 1 << (32*W32)
        if u != vals[r]:
            return False, r
    return True, None
random.seed(1)
print(check(16, 256, 33, 3, 8192))
print(check(64, 4, 56, 4, 23))
print(check(1, 2048, 33, 4, 65536))
