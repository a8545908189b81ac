"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

Holds NO method arithmetic (no windows, codes, Hadamards, LCGs): only numpy
`default_rng` draws with fixed seeds, so both the oracle and the CUDA path can
consume byte-identical inputs (SURVEY §8(d) seed plan):
    packed tiles of layer l : 1000 + l     x (batch column b): 2000 (+ b)
    input signs S_n         : 3000         output signs S_m  : 3001
    HYB LUT                 : 4000         Gaussian sources   : 5000
Any kT-bit string is a valid tail-biting trellis walk, so uniform
random bytes are valid packed weights; decode cost is data-independent.
"""
import numpy as np

TILE = 16


def tile_bytes(k, T=256):
    return k * T // 8


def random_tiles(m, n, k, seed=1000, Tx=TILE, Ty=TILE):
    """uint8 (m/Tx, n/Ty, 32k): logical tail-biting tile streams (T = Tx Ty = 256), MSB-first."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, 256, size=(m // Tx, n // Ty, tile_bytes(k)), dtype=np.uint8)


def random_x(B, n, seed=2000):
    """(B, n) float32 i.i.d. N(0, 1) activations."""
    rng = np.random.default_rng(seed)
    return rng.standard_normal((B, n)).astype(np.float32)


def random_sign_bytes(n, seed):
    """ceil(n/8) bytes of Bernoulli(1/2) sign bits (bit set = negative)."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, 256, size=(n + 7) // 8, dtype=np.uint8)


def gaussian_lut(Q, seed=4000):
    """A (2^Q, 2) binary16 table of i.i.d. N(0, 1) draws (any fp16 table is a valid HYB
    LUT; the k-means LUT of P:309 lives in oracle.codes)."""
    rng = np.random.default_rng(seed)
    return rng.standard_normal((1 << Q, 2)).astype(np.float16).view(np.uint16)


def gaussian_table(nbits, seed=4001):
    """A (2^nbits,) binary16 table of i.i.d. N(0, 1) draws: the 1-D codebook of HYB with V = 1
     or the lookup-only code's 2^L table ("~ N(0, 1)")."""
    rng = np.random.default_rng(seed)
    return rng.standard_normal(1 << nbits).astype(np.float16).view(np.uint16)


def gaussian_source(nseq, T, seed=5000):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((nseq, T))


def synthetic_hessian(n, N=None, rho=0.9, damp=1e-2, seed=6000):
    """A proxy Hessian H = X^T X / N + damp * mean(diag) I of N activation rows drawn from an AR(1)
    Gaussian (correlation rho^|i-j|): PSD, correlated like real layer inputs (no trained weights or
    datasets are available here; reading R21)."""
    rng = np.random.default_rng(seed)
    N = N or 4 * n
    Z = rng.standard_normal((N, n))
    X = np.empty_like(Z)
    X[:, 0] = Z[:, 0]
    for i in range(1, n):
        X[:, i] = rho * X[:, i - 1] + np.sqrt(1 - rho * rho) * Z[:, i]
    H = X.T @ X / N
    return H + damp * np.mean(np.diag(H)) * np.eye(n)
