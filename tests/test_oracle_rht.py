"""Pins for oracle.hadamard / oracle.rht: H H^T = n I, skew Paley structure, structured == dense,
orthogonality and invertibility of the RHT, the incoherence bound of P:98."""
import numpy as np
import pytest

from oracle import hadamard, rht


@pytest.mark.parametrize("n", [1, 2, 4, 16, 128, 1024])
def test_sylvester_orthogonal(n):
    H = hadamard.sylvester(n)
    assert (H @ H.T == n * np.eye(n)).all()
    assert (H == H.T).all()


@pytest.mark.parametrize("b", [4, 8, 12, 20, 28, 44, 108, 344])
def test_paley_orders(b):
    H = hadamard.hadamard_b(b)
    assert set(np.unique(H)) <= {-1, 1}
    assert (H @ H.T == b * np.eye(b, dtype=np.int64)).all()
    assert (H + H.T == 2 * np.eye(b, dtype=np.int64)).all()           # Paley I is skew-type


def test_factor_rule_llama_dims():
    assert hadamard.factor(4096) == (1, 12)
    assert hadamard.factor(8192) == (1, 13)
    assert hadamard.factor(11008) == (344, 5)        # 11008 = 344 * 32 (P:855-857 reading R7)
    assert hadamard.factor(28672) == (28, 10)        # 28672 = 28 * 1024
    assert hadamard.factor(256) == (1, 8)
    assert hadamard.factor(5120) == (20, 8)          # Llama-2-13B hidden (q = 19)
    assert hadamard.factor(13824) == (108, 7)        # Llama-2-13B MLP (q = 107)
    assert hadamard.factor(16 * 9) == (72, 1)        # q = 71: smallest order with n/b a power of two


def test_factor_rejects_unsupported():
    with pytest.raises(ValueError):
        hadamard.factor(3 * 5 * 7)


@pytest.mark.parametrize("n", [12 * 4, 28 * 8, 344 * 2, 64, 1024, 20 * 16])
def test_structured_equals_dense(n):
    rng = np.random.default_rng(n)
    x = rng.standard_normal((3, n))
    H = hadamard.hadamard(n).astype(np.float64)
    assert np.allclose(rht.apply_hadamard(x, n), x @ H.T, rtol=0, atol=1e-9)
    assert np.allclose(rht.apply_hadamard(x, n, transpose=True), x @ H, rtol=0, atol=1e-9)
    assert (H @ H.T == n * np.eye(n)).all()


@pytest.mark.parametrize("n", [256, 4096, 11008, 28672])
def test_rht_orthogonal_and_invertible(n):
    rng = np.random.default_rng(1)
    x = rng.standard_normal((2, n))
    s = rng.integers(0, 256, (n + 7) // 8, dtype=np.uint8)
    xt = rht.rht_forward(x, s, n)
    assert np.allclose(np.linalg.norm(xt, axis=1), np.linalg.norm(x, axis=1), rtol=1e-12)
    assert np.allclose(rht.rht_inverse(xt, s, n), x, atol=1e-12)


def test_sign_bits_lsb_first():
    s = np.array([0b00000101, 0b10000000], dtype=np.uint8)
    assert list(rht.signs_from_bits(s, 16)) == [-1, 1, -1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, -1]


def test_rht_incoherence_bound():
    """after the RHT, mu_W~ <= 2 log(4 m n / delta) w.h.p. (checked with delta = 0.01)
    on a matrix with a huge outlier that is very coherent before processing."""
    rng = np.random.default_rng(5)
    m, n = 64, 128
    W = rng.standard_normal((m, n))
    W[3, 7] = 500.0
    sm = rng.integers(0, 256, m // 8, dtype=np.uint8)
    sn = rng.integers(0, 256, n // 8, dtype=np.uint8)
    Wt = rht.rht_matrix(W, sm, sn)
    assert rht.incoherence_mu(W) > 30
    assert rht.incoherence_mu(Wt) <= 2 * np.log(4 * m * n / 0.01)
    assert np.isclose(np.linalg.norm(Wt), np.linalg.norm(W))       # orthogonal conjugation


def test_rht_matrix_consistent_with_vector_rht():
    """W x = S_m H_m^T (W~ x~) with x~ = RHT(x): the relation the inference path relies on."""
    rng = np.random.default_rng(6)
    m, n = 48, 56
    W = rng.standard_normal((m, n))
    x = rng.standard_normal((1, n))
    sm = rng.integers(0, 256, m // 8, dtype=np.uint8)
    sn = rng.integers(0, 256, n // 8, dtype=np.uint8)
    Wt = rht.rht_matrix(W, sm, sn)
    y = rht.rht_inverse(rht.rht_forward(x, sn, n) @ Wt.T, sm, m)
    assert np.allclose(y, x @ W.T, atol=1e-10)
