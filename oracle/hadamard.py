"""Hadamard matrices for the RHT.  (oracle; test infrastructure only)

Paper passages:
  P:96-97   RHT uses V_k, a k x k Hadamard matrix, with a random sign vector S_k.
  P:855-857 "We use Hadamard matrices from Neil Sloane's website."  That table is not
            available offline; reading R7: for n = b * 2^a we use
            H_n = kron(H_b, H_{2^a}) (row index i = i_b * 2^a + i_a), H_{2^a} the
            Sylvester matrix H[i, j] = (-1)^popcount(i & j), and H_b the Paley-I
            (skew) Hadamard matrix of order b = q + 1 for a prime power q = 3 mod 4:
              H_b = I + [[0, 1^T], [-1, Jq]],  Jq[i, j] = chi(g_i - g_j),
            chi the quadratic character of GF(q), row/col 0 the point at infinity,
            g_i the i-th field element.  Field elements are indexed by their base-p
            digits (c0 + c1 p + c2 p^2 <-> c0 + c1 x + c2 x^2).  GF(27) = GF(3)[x]/(x^3+2x+1),
            GF(343) = GF(7)[x]/(x^3+4).  b is the smallest supported order with n/b a
            power of two (b = 1 when n is a power of two).
"""
import numpy as np


def is_pow2(n):
    return n >= 1 and (n & (n - 1)) == 0


def _is_prime(q):
    if q < 2:
        return False
    d = 2
    while d * d <= q:
        if q % d == 0:
            return False
        d += 1
    return True


# prime-power fields we support beyond prime q: q -> (p, modulus coefficients c0, c1, c2 of x^3 + c2 x^2 + c1 x + c0)
PRIME_POWER_FIELDS = {27: (3, (1, 2, 0)), 343: (7, (4, 0, 0))}
MAX_PALEY_ORDER = 1024


def supported_orders():
    out = [1]
    for q in range(3, MAX_PALEY_ORDER):
        if q % 4 == 3 and (_is_prime(q) or q in PRIME_POWER_FIELDS):
            out.append(q + 1)
    return sorted(out)


def factor(n):
    """(b, a) with n = b * 2^a, b the smallest supported Paley order (or 1)."""
    for b in supported_orders():
        if n % b == 0 and is_pow2(n // b):
            return b, (n // b).bit_length() - 1
    raise ValueError(f"no supported Hadamard order for n={n}")


def sylvester(n):
    """H[i, j] = (-1)^popcount(i & j), the Sylvester construction of order 2^a."""
    assert is_pow2(n)
    i = np.arange(n)
    pc = np.zeros((n, n), dtype=np.int64)
    x = i[:, None] & i[None, :]
    while x.any():
        pc += x & 1
        x = x >> 1
    return np.where(pc % 2 == 0, 1, -1).astype(np.int64)


def _field(q):
    """Elements as digit tuples, with subtraction and multiplication (plain polynomial arithmetic)."""
    if _is_prime(q):
        p, deg, mod = q, 1, None
    else:
        p, mod = PRIME_POWER_FIELDS[q]
        deg = 3
    elems = []
    for i in range(q):
        d, v = [], i
        for _ in range(deg):
            d.append(v % p)
            v //= p
        elems.append(tuple(d))

    def sub(u, v):
        return tuple((a - b) % p for a, b in zip(u, v))

    def mul(u, v):
        if deg == 1:
            return ((u[0] * v[0]) % p,)
        prod = [0] * 5
        for i, a in enumerate(u):
            for j, b in enumerate(v):
                prod[i + j] += a * b
        # reduce with x^3 = -(c2 x^2 + c1 x + c0)
        c0, c1, c2 = mod
        for e in (4, 3):
            t = prod[e]
            prod[e] = 0
            prod[e - 3] -= t * c0
            prod[e - 2] -= t * c1
            prod[e - 1] -= t * c2
        return tuple(c % p for c in prod[:3])

    return elems, sub, mul


def paley1(b):
    """Paley-I Hadamard matrix of order b = q + 1 (q = 3 mod 4, prime or in PRIME_POWER_FIELDS)."""
    q = b - 1
    elems, sub, mul = _field(q)
    zero = elems[0]
    squares = {mul(e, e) for e in elems if e != zero}
    index = {e: i for i, e in enumerate(elems)}

    def chi(e):
        if e == zero:
            return 0
        return 1 if e in squares else -1

    Jq = np.array([[chi(sub(elems[i], elems[j])) for j in range(q)] for i in range(q)], dtype=np.int64)
    S = np.zeros((b, b), dtype=np.int64)
    S[0, 1:] = 1
    S[1:, 0] = -1
    S[1:, 1:] = Jq
    del index
    return np.eye(b, dtype=np.int64) + S


def hadamard_b(b):
    return np.ones((1, 1), dtype=np.int64) if b == 1 else paley1(b)


def hadamard(n):
    """Dense integer H_n = kron(H_b, H_{2^a}) (small n only; used to pin the structured RHT)."""
    b, a = factor(n)
    return np.kron(hadamard_b(b), sylvester(1 << a))
