"""QTIP node-value codes: 1MAD (Alg. 1), 3INST (Alg. 2), HYB (Alg. 3).  (oracle; test infrastructure only)

Paper passages:
  P:254-260, P:269-281  1MAD: x <- (a x + b) mod 2^32; sum the four bytes;
                        (s - 510)/147.8; a = 34038481, b = 76625530.
  P:262-267, P:283-296  3INST: x <- (a x + b) mod 2^32;
                        m <- reinterpret(m) << 16 + reinterpret(m);
                        x <- (x & 0b1000_1111_1111_1111_1000_1111_1111_1111) XOR m;
                        return f16(x & 0xFFFF) + f16(x >> 16);
                        a = 89226354, b = 64248484, m = 0.922 (fp16).
  P:298-321             HYB: x <- x*x + x mod 2^32; v <- C[(x >> (15-Q)) & (2^Q - 1)];
                        v <- v XOR (x & (1 << 15)); "two sign flip" also XORs bit 31.
  P:309                 LUT initialised by k-means on 2-D i.i.d. Gaussian samples.
  P:607-609             HYB with a 1-D codebook (Q = 6, V = 1): the same hash, index and sign
                        flip with a 2^Q-entry table of single values (v XOR (x & (1 << 15))).
  P:751-798             lookup-only code: the value of state x is LUT[x], a 2^L-entry table
                        (L = 14, V = 1, T_x = 32, T_y = 8; "~ N(0, 1)", tunable).

Output precision readings:
  * 1MAD returns the IEEE binary16 round-to-nearest-even of the exact rational
    (s - 510)/147.8 (the paper's 16-bit GPU datapath; Alg. 1 states no rounding).
  * 3INST returns binary16 RNE of the exact sum m1 + m2 (footnote P:265: summed as
    two FP16s, i.e. one fp16 addition).
  * HYB: a LUT entry is the 32-bit word (bits16(c0) << 16) | bits16(c1), c0 the value
    for the earlier sequence position.  Bit 15 then is the sign of c1, so the XOR of
    Alg. 3 flips "the sign of the second entry" exactly as the prose of P:304 says.
Arithmetic is exact Python/numpy integer arithmetic; fp16 rounding is done from
exact Fractions (`fp16_rne`) or from exact float64 values via one numpy cast.
"""
from fractions import Fraction
import numpy as np

# Constants exactly as printed in the paper.
A_1MAD, B_1MAD = 34038481, 76625530
A_3INST, B_3INST = 89226354, 64248484
M_3INST = Fraction("0.922")
MASK_3INST = 0b10001111111111111000111111111111
MOD32 = 1 << 32


# ---------------------------------------------------------------- binary16
def fp16_rne(v):
    """Round an exact rational to IEEE binary16 (round-to-nearest-even); returns the
    16-bit pattern as int.  Written out from the IEEE definition."""
    v = Fraction(v)
    sign = 0x8000 if v < 0 else 0
    a = -v if v < 0 else v
    if a == 0:
        return sign
    # e = floor(log2 a)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    if e < -14:                      # subnormal range: ulp 2^-24
        ulp = Fraction(1, 1 << 24)
        q = a / ulp
        n = q.numerator // q.denominator
        rem = q - n
        if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and n % 2 == 1):
            n += 1
        return sign | n              # n == 1024 encodes the smallest normal
    ulp = Fraction(2) ** (e - 10)
    q = a / ulp
    n = q.numerator // q.denominator
    rem = q - n
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and n % 2 == 1):
        n += 1
    if n == 2048:
        n = 1024
        e += 1
    if e > 15:
        return sign | 0x7C00         # overflow -> inf
    return sign | ((e + 15) << 10) | (n - 1024)


def fp16_value(bits):
    """Exact value (Fraction) of a finite binary16 pattern."""
    bits = int(bits) & 0xFFFF
    s = -1 if bits & 0x8000 else 1
    e = (bits >> 10) & 0x1F
    f = bits & 0x3FF
    if e == 0x1F:
        raise ValueError("inf/nan")
    if e == 0:
        return s * Fraction(f, 1 << 24)
    return s * (1 + Fraction(f, 1024)) * Fraction(2) ** (e - 15)


def f16_to_f64(bits):
    """Vectorised exact binary16 -> float64 (numpy cast is exact for finite values)."""
    return np.asarray(bits, dtype=np.uint16).view(np.float16).astype(np.float64)


# ---------------------------------------------------------------- LCG
def lcg(x, a, b):
    """(a x + b) mod 2^32, exact on uint64 arrays or Python ints."""
    if isinstance(x, (int, np.integer)):
        return (a * int(x) + b) % MOD32
    x = np.asarray(x, dtype=np.uint64)
    return (np.uint64(a) * x + np.uint64(b)) & np.uint64(MOD32 - 1)   # a*x < 2^64 since a < 2^27, x < 2^32


# ---------------------------------------------------------------- 1MAD (Alg. 1)
def byte_sum(y):
    y = np.asarray(y, dtype=np.uint64)
    return ((y & 255) + ((y >> 8) & 255) + ((y >> 16) & 255) + ((y >> 24) & 255)).astype(np.int64)


_ONEMAD_TABLE = None


def onemad_value_from_sum(s):
    """binary16 RNE of the exact rational (s - 510)/147.8, for every byte sum s in [0, 1020]."""
    global _ONEMAD_TABLE
    if _ONEMAD_TABLE is None:
        _ONEMAD_TABLE = np.array([fp16_rne(Fraction(t - 510) / Fraction("147.8")) for t in range(1021)],
                                 dtype=np.uint16)
    return _ONEMAD_TABLE[np.asarray(s, dtype=np.int64)]


def decode_1mad(x, a=A_1MAD, b=B_1MAD):
    """Alg. 1.  x: states (ints / array).  Returns binary16 bit patterns (uint16)."""
    y = lcg(np.asarray(x, dtype=np.uint64), a, b)
    return onemad_value_from_sum(byte_sum(y))


# ---------------------------------------------------------------- 3INST (Alg. 2)
def magic_word_3inst(m=M_3INST):
    """reinterpret(m) << 16 + reinterpret(m)  (read as bitwise OR of the two halves)."""
    mb = fp16_rne(m)
    return (mb << 16) | mb


def inst3_halves(x, a=A_3INST, b=B_3INST, m=M_3INST):
    """The masked/XORed word of P:291 split into its two binary16 patterns (m1 = low, m2 = high)."""
    y = lcg(np.asarray(x, dtype=np.uint64), a, b)
    z = (y & np.uint64(MASK_3INST)) ^ np.uint64(magic_word_3inst(m))
    return (z & np.uint64(0xFFFF)).astype(np.uint16), (z >> np.uint64(16)).astype(np.uint16)


def decode_3inst(x, a=A_3INST, b=B_3INST, m=M_3INST):
    """Alg. 2: binary16 RNE of m1 + m2.  Returns uint16 bit patterns.
    m1 + m2 of two binary16 values is exact in float64; the single cast rounds RNE."""
    m1, m2 = inst3_halves(x, a, b, m)
    s = f16_to_f64(m1) + f16_to_f64(m2)
    return s.astype(np.float16).view(np.uint16)


def decode_3inst_exact(x, a=A_3INST, b=B_3INST, m=M_3INST):
    """Scalar Fraction form of Alg. 2 (for pins): returns (z, m1+m2 exact, fp16 bits)."""
    y = lcg(int(x), a, b)
    z = (y & MASK_3INST) ^ magic_word_3inst(m)
    tot = fp16_value(z & 0xFFFF) + fp16_value(z >> 16)
    return z, tot, fp16_rne(tot)


# ---------------------------------------------------------------- HYB (Alg. 3)
def hyb_hash(x):
    x = np.asarray(x, dtype=np.uint64)
    return (x * x + x) & np.uint64(MOD32 - 1)     # x < 2^32 -> x*x < 2^64


def hyb_index(h, Q):
    return ((np.asarray(h, dtype=np.uint64) >> np.uint64(15 - Q)) & np.uint64((1 << Q) - 1)).astype(np.int64)


def decode_hyb(x, lut, Q, two_sign=False):
    """Alg. 3.  lut: uint16 (2^Q, 2) binary16 patterns, column 0 = c0
    (earlier position), column 1 = c1.  Returns uint16 (..., 2): (value at 2t, value at 2t+1)."""
    lut = np.asarray(lut, dtype=np.uint16)
    h = hyb_hash(x)
    idx = hyb_index(h, Q)
    word = (lut[idx, 0].astype(np.uint64) << np.uint64(16)) | lut[idx, 1].astype(np.uint64)
    flip = h & np.uint64(1 << 15)
    if two_sign:
        flip = flip | (h & np.uint64(1 << 31))
    word = word ^ flip
    return np.stack([(word >> np.uint64(16)).astype(np.uint16), (word & np.uint64(0xFFFF)).astype(np.uint16)],
                    axis=-1)


def decode_hyb1(x, lut1, Q):
    """HYB with a 1-D codebook (V = 1): Alg. 3's hash and index, lut1 uint16 (2^Q,)
    binary16 patterns; the value's sign bit is XORed with bit 15 of the hash (P:317 with a
    16-bit v).  Returns uint16 (...)."""
    lut1 = np.asarray(lut1, dtype=np.uint16)
    h = hyb_hash(x)
    idx = hyb_index(h, Q)
    return (lut1[idx].astype(np.uint64) ^ (h & np.uint64(1 << 15))).astype(np.uint16)


def decode_lut(x, lut):
    """Lookup-only code: the value of state x (L bits) is lut[x]; lut uint16
    (2^L,) binary16 patterns.  Returns uint16 (...)."""
    lut = np.asarray(lut, dtype=np.uint16)
    return lut[np.asarray(x, dtype=np.int64)]


def kmeans_lut(Q, seed=4000, n_samples=1 << 18, iters=40):
    """k-means (Lloyd) with 2^Q centroids on i.i.d. N(0, I_2) samples.
    Deterministic given seed; init = a random subset of the samples; an empty cluster
    is re-seeded at the sample farthest from its centroid.  Returns uint16 (2^Q, 2)."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n_samples, 2))
    K = 1 << Q
    C = X[rng.choice(n_samples, K, replace=False)].copy()
    for _ in range(iters):
        # assignment (chunked to bound memory)
        lab = np.empty(n_samples, dtype=np.int64)
        dmin = np.empty(n_samples)
        for s in range(0, n_samples, 1 << 14):
            Xs = X[s:s + (1 << 14)]
            # squared distances ||x||^2 - 2 x.c + ||c||^2
            d = (Xs ** 2).sum(1)[:, None] - 2.0 * Xs @ C.T + (C ** 2).sum(1)[None, :]
            lab[s:s + (1 << 14)] = d.argmin(1)
            dmin[s:s + (1 << 14)] = d.min(1)
        cnt = np.bincount(lab, minlength=K)
        for d in range(2):
            C[:, d] = np.where(cnt > 0, np.bincount(lab, weights=X[:, d], minlength=K) / np.maximum(cnt, 1), C[:, d])
        for e in np.flatnonzero(cnt == 0):
            far = int(dmin.argmax())
            C[e] = X[far]
            dmin[far] = 0.0
    return C.astype(np.float16).view(np.uint16).reshape(K, 2)


# ---------------------------------------------------------------- tables & moments
def code_table(code, L, lut=None, Q=9, two_sign=False):
    """float64 values of the code for every state 0..2^L-1: shape (2^L,) or (2^L, 2)."""
    xs = np.arange(1 << L, dtype=np.uint64)
    if code == "1mad":
        return f16_to_f64(decode_1mad(xs))
    if code == "3inst":
        return f16_to_f64(decode_3inst(xs))
    if code == "hyb":
        return f16_to_f64(decode_hyb(xs, lut, Q, two_sign))
    if code == "hyb1":
        return f16_to_f64(decode_hyb1(xs, lut, Q))
    if code == "lut":
        return f16_to_f64(decode_lut(xs, lut))
    raise ValueError(code)


def distortion_rate_bound(k):
    """D_R = 2^{-2k} for a unit-variance Gaussian source (Table 1 'D_R' = 0.063 at k=2)."""
    return 2.0 ** (-2 * k)


def neighbor_correlation(table, L, k, V=1):
    """Fig. 3: Pearson correlation of (last value of s, first value of s')
    over every edge (s, s') of the (L,k,V) bitshift trellis."""
    kv = k * V
    s = np.repeat(np.arange(1 << L), 1 << kv)
    c = np.tile(np.arange(1 << kv), 1 << L)
    t = ((s << kv) % (1 << L)) + c
    tab = np.asarray(table)
    a = tab[s] if tab.ndim == 1 else tab[s, -1]
    b = tab[t] if tab.ndim == 1 else tab[t, 0]
    if a.std() == 0 or b.std() == 0:
        return 0.0
    return float(np.corrcoef(a, b)[0, 1])
