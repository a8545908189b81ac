"""BlockLDLQ with QTIP as its rounding step (Algorithm 5).  (oracle; test infrastructure only)

Paper passages:
  P:821-823  QTIP is "a drop-in replacement for vector quantization in BlockLDLQ": the step
             Q(W + (W - W^) A) is unchanged; Q rounds T_x rows x T_y columns as one sequence.
  Alg. 5     W^ <- 0;  L D L^T <- T_y-block LDL decomposition of H;  A <- L - I;
             for j = n/T_y - 1 down to 0:
                 x <- W[:, jT_y:(j+1)T_y] + (W[:, jT_y:] - W^[:, jT_y:]) A[jT_y:, jT_y:(j+1)T_y]
                 x <- x.reshape(m/T_x, T_x T_y)
                 x^ <- Viterbi(x, (L, k, V) bitshift trellis, C)  (row-wise)
                 W^[:, jT_y:(j+1)T_y] <- x^.reshape(m, T_y)

Readings: the "Viterbi" of a row is the tail-biting Algorithm 4 (the paper's
quantizer for every experiment); the T_y-block LDL factor L is unit lower block-triangular with H =
L D L^T, D block diagonal, so A = L - I is strictly lower block-triangular and the loop (right to left)
feeds back the errors of the blocks already quantized (rows below block j).  Written in float64 with
plain numpy linear algebra, step by step.
"""
import numpy as np

from . import viterbi


def block_ldl(H, Ty):
    """T_y-block LDL decomposition H = L D L^T (L unit lower block-triangular, D block diagonal),
    by the block recurrence D_j = H_jj - sum_{k<j} L_jk D_k L_jk^T,
    L_ij = (H_ij - sum_{k<j} L_ik D_k L_jk^T) D_j^{-1} (i > j).  Returns (L, D) as n x n arrays."""
    H = np.asarray(H, dtype=np.float64)
    n = H.shape[0]
    nb = n // Ty
    Lm = np.eye(n)
    D = np.zeros((n, n))
    blk = lambda a: slice(a * Ty, (a + 1) * Ty)  # noqa: E731
    for j in range(nb):
        Dj = H[blk(j), blk(j)].copy()
        for k in range(j):
            Dj -= Lm[blk(j), blk(k)] @ D[blk(k), blk(k)] @ Lm[blk(j), blk(k)].T
        D[blk(j), blk(j)] = Dj
        Djinv = np.linalg.inv(Dj)
        for i in range(j + 1, nb):
            Sij = H[blk(i), blk(j)].copy()
            for k in range(j):
                Sij -= Lm[blk(i), blk(k)] @ D[blk(k), blk(k)] @ Lm[blk(j), blk(k)].T
            Lm[blk(i), blk(j)] = Sij @ Djinv
    return Lm, D


def blockldlq(W, H, Tx, Ty, L, k, V, code_table, quantize=None):
    """Algorithm 5.  code_table: float64 values of the code over the 2^L states ((2^L,) or (2^L, V)).
    quantize(S) -> (states (nseq, T/V), costs) rounds sequences S (nseq, T); default: Algorithm 4 in
    float64 (viterbi.tailbite_encode_batch).  Returns (W^, states per block column (n/Ty, m/Tx, T/V))."""
    W = np.asarray(W, dtype=np.float64)
    m, n = W.shape
    if quantize is None:
        quantize = lambda S: viterbi.tailbite_encode_batch(S, L, k, V, code_table)  # noqa: E731
    tab = np.asarray(code_table, dtype=np.float64).reshape(1 << L, V)
    Lm, _ = block_ldl(H, Ty)
    A = Lm - np.eye(n)
    What = np.zeros((m, n))
    walks = [None] * (n // Ty)
    for j in range(n // Ty - 1, -1, -1):
        c0, c1 = j * Ty, (j + 1) * Ty
        x = W[:, c0:c1] + (W[:, c0:] - What[:, c0:]) @ A[c0:, c0:c1]
        xs = x.reshape(m // Tx, Tx * Ty)                      # T_x rows of T_y columns per sequence
        st, _ = quantize(xs)
        xh = tab[np.asarray(st, dtype=np.int64)].reshape(m // Tx, Tx * Ty)
        What[:, c0:c1] = xh.reshape(m, Ty)
        walks[j] = np.asarray(st)
    return What, np.stack(walks)


def proxy_loss(W, What, H):
    """tr((W - W^) H (W - W^)^T): the proxy objective BlockLDLQ minimises."""
    E = np.asarray(W, dtype=np.float64) - np.asarray(What, dtype=np.float64)
    return float(np.trace(E @ np.asarray(H, dtype=np.float64) @ E.T))


# the synthetic proxy Hessian is an input recipe (no method arithmetic): it lives in synth/, shared
# by the oracle's tests and the GPU tests
from synth import synthetic_hessian  # noqa: E402,F401
