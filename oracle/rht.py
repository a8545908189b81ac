"""Random Hadamard transform (RHT) on activations.  (oracle; test infrastructure only)

Paper passages:
  P:96-97  W~ <- V_m S_m W S_n V_n^T  (V_k a Hadamard matrix, S_k a random sign vector).
  P:98     with probability >= 1 - delta, mu_W~ = 2 log(4 m n / delta).
  P:90-93  Definition 2.1 (mu-incoherence).

Reading R8: with orthonormal H_k = V_k / sqrt(k) and the stored
RHT-domain matrix W~, the layer computes
    y = W x = S_m H_m^T  W~  H_n S_n x,
so the inference path is  x~ = H_n (S_n . x) / sqrt(n)   (RHT in)
                          y  = S_m . (H_m^T y~) / sqrt(m) (RHT out; H^T matters for
                                                           the skew Paley factors).
Sign vectors are bit-packed: element i is negative iff bit (i & 7) of byte i >> 3 is set.
"""
import numpy as np

from . import hadamard


def signs_from_bits(sign_bytes, n):
    b = np.asarray(sign_bytes, dtype=np.uint8)
    bits = np.unpackbits(b, bitorder="little")[:n]
    return np.where(bits == 1, -1.0, 1.0)


def apply_hadamard(x, n, transpose=False):
    """Integer H_n (or H_n^T) applied to the last axis of x, using the Kronecker structure
    H_n = H_b (x) H_2 (x) ... (x) H_2 factor by factor (the definition of the product)."""
    b, a = hadamard.factor(n)
    x = np.asarray(x, dtype=np.float64)
    lead = x.shape[:-1]
    t = x.reshape(lead + (b,) + (2,) * a)
    Hb = hadamard.hadamard_b(b).astype(np.float64)
    if transpose:
        Hb = Hb.T
    ax = len(lead)
    t = np.moveaxis(np.tensordot(Hb, t, axes=([1], [ax])), 0, ax)
    for d in range(a):
        axd = ax + 1 + d
        t0 = np.take(t, 0, axis=axd)
        t1 = np.take(t, 1, axis=axd)
        t = np.stack([t0 + t1, t0 - t1], axis=axd)
    return t.reshape(lead + (n,))


def rht_forward(x, sign_bytes, n):
    """x~ = H_n (S_n . x) / sqrt(n) over the last axis."""
    s = signs_from_bits(sign_bytes, n)
    return apply_hadamard(np.asarray(x, dtype=np.float64) * s, n) / np.sqrt(n)


def rht_inverse(y, sign_bytes, n):
    """S_n . (H_n^T y) / sqrt(n) over the last axis (inverse of rht_forward)."""
    s = signs_from_bits(sign_bytes, n)
    return apply_hadamard(np.asarray(y, dtype=np.float64), n, transpose=True) * s / np.sqrt(n)


def incoherence_mu(W):
    """Definition 2.1: smallest mu with max|W_ij| <= mu ||W||_F / sqrt(mn)."""
    W = np.asarray(W, dtype=np.float64)
    m, n = W.shape
    return float(np.abs(W).max() * np.sqrt(m * n) / np.linalg.norm(W))


def rht_matrix(W, sign_m, sign_n):
    """W~ = H_m S_m W S_n H_n^T / sqrt(mn) (P:97 with orthonormal Hadamards)."""
    m, n = W.shape
    sm = signs_from_bits(sign_m, m)
    sn = signs_from_bits(sign_n, n)
    A = apply_hadamard((W * sn[None, :]), n)            # rows: (H_n S_n w_i)  == (W S_n H_n^T)_i
    A = apply_hadamard((A * sm[:, None]).T, m).T        # H_m S_m (...)
    return A / np.sqrt(m * n)
