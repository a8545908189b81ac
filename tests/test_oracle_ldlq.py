"""Pins of the oracle's BlockLDLQ (Algorithm 5)."""
import numpy as np

import synth
from oracle import codes, ldlq, viterbi

L, K, V = 12, 2, 1          # a small trellis keeps the CPU DP fast (Table 3's L = 12)


def _table():
    t = codes.f16_to_f64(synth.gaussian_table(L, seed=4100))
    return t / t.std()


def test_block_ldl_factorises_h():
    H = ldlq.synthetic_hessian(64, seed=1)
    for Ty in (1, 4, 8, 16):
        Lm, D = ldlq.block_ldl(H, Ty)
        assert np.allclose(Lm @ D @ Lm.T, H, atol=1e-10, rtol=0)
        for i in range(64 // Ty):
            assert np.array_equal(Lm[i * Ty:(i + 1) * Ty, i * Ty:(i + 1) * Ty], np.eye(Ty))       # unit diagonal blocks
            assert not np.any(Lm[i * Ty:(i + 1) * Ty, (i + 1) * Ty:])                            # lower block-triangular
            assert not np.any(D[i * Ty:(i + 1) * Ty, (i + 1) * Ty:])                             # block diagonal
            assert np.all(np.linalg.eigvalsh(D[i * Ty:(i + 1) * Ty, i * Ty:(i + 1) * Ty]) > 0)


def test_identity_hessian_reduces_to_blockwise_quantization():
    """H = I: L = I, A = 0, so every block column is rounded on its own (Algorithm 4 per sequence)."""
    rng = np.random.default_rng(2)
    m, n, Tx, Ty = 32, 32, 16, 16
    W = rng.standard_normal((m, n))
    tab = _table()
    What, _ = ldlq.blockldlq(W, np.eye(n), Tx, Ty, L, K, V, tab)
    for j in range(n // Ty):
        S = W[:, j * Ty:(j + 1) * Ty].reshape(m // Tx, Tx * Ty)
        st, _ = viterbi.tailbite_encode_batch(S, L, K, V, tab)
        assert np.array_equal(What[:, j * Ty:(j + 1) * Ty], tab[st].reshape(m, Ty))


def test_ldlq_error_identity():
    """With E = W - W^ and H = L D L^T, tr(E H E^T) = sum_j ||(E L)_j||^2_{D_j}, and (E L)_j = x_j - W^_j
    is exactly block j's rounding error: the feedback term makes the proxy loss the D-weighted sum of
    the per-block rounding errors (a sign or index slip in the feedback breaks it)."""
    rng = np.random.default_rng(3)
    m, n, Tx, Ty = 16, 64, 16, 16
    W = rng.standard_normal((m, n))
    H = ldlq.synthetic_hessian(n, seed=4)
    tab = _table()
    What, _ = ldlq.blockldlq(W, H, Tx, Ty, L, K, V, tab)
    Lm, D = ldlq.block_ldl(H, Ty)
    A = Lm - np.eye(n)
    tot = 0.0
    for j in range(n // Ty):
        c0, c1 = j * Ty, (j + 1) * Ty
        x = W[:, c0:c1] + (W[:, c0:] - What[:, c0:]) @ A[c0:, c0:c1]      # the input Alg. 5 rounded
        r = x - What[:, c0:c1]
        tot += float(np.trace(r @ D[c0:c1, c0:c1] @ r.T))
    assert np.isclose(tot, ldlq.proxy_loss(W, What, H), rtol=1e-9, atol=1e-9)


def test_feedback_lowers_the_proxy_loss():
    """On correlated (AR(1)) synthetic Hessians the error feedback beats rounding each block alone."""
    rng = np.random.default_rng(5)
    m, n, Tx, Ty = 16, 64, 16, 16
    tab = _table()
    wins = 0
    for s in range(3):
        W = rng.standard_normal((m, n))
        H = ldlq.synthetic_hessian(n, rho=0.95, seed=10 + s)
        Wl, _ = ldlq.blockldlq(W, H, Tx, Ty, L, K, V, tab)
        Wd, _ = ldlq.blockldlq(W, np.eye(n), Tx, Ty, L, K, V, tab)       # feedback off
        wins += ldlq.proxy_loss(W, Wl, H) < ldlq.proxy_loss(W, Wd, H)
    assert wins == 3


def test_sequences_are_tx_rows_of_ty_columns():
    """x.reshape(m / T_x, T_x T_y): the rounding sees T_x consecutive rows of the block column, row-major
    (P:833), so with T_x = 32, T_y = 8 a sequence is a 32 x 8 block in row order."""
    rng = np.random.default_rng(6)
    m, n, Tx, Ty = 64, 16, 32, 8
    W = rng.standard_normal((m, n))
    tab = _table()
    seen = []

    def q(S):
        seen.append(S.copy())
        return viterbi.tailbite_encode_batch(S, L, K, V, tab)
    ldlq.blockldlq(W, np.eye(n), Tx, Ty, L, K, V, tab, quantize=q)
    assert np.array_equal(seen[0][1], W[32:64, 8:16].reshape(-1))     # j = 1 first, second block of rows
    assert np.array_equal(seen[1][0], W[0:32, 0:8].reshape(-1))
