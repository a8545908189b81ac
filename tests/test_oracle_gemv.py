"""Pins for oracle.gemv: vectorised dense decode == per-weight scalar definition (windows +
exact codes), matvec == explicit dense S_m H_m^T W~ H_n S_n product, special cases."""
import numpy as np
import pytest

import synth
from oracle import codes, gemv, hadamard, rht, trellis


def _scalar_decode(tiles, p):
    """Per weight, straight from the definitions: window(bits, t) -> code -> binary16 value."""
    mt, nt, _ = tiles.shape
    W = np.zeros((mt * 16, nt * 16))
    for I in range(mt):
        for J in range(nt):
            bits = trellis.bits_from_bytes(tiles[I, J], p.k * 256)
            for t in range(256 // p.V):
                s = trellis.window(bits, t, p.L, p.k, p.V, tail_biting=True)
                if p.code == "3inst":
                    vals = [float(codes.fp16_value(codes.decode_3inst_exact(s)[2]))]
                elif p.code == "1mad":
                    y = codes.lcg(s, codes.A_1MAD, codes.B_1MAD)
                    ssum = sum((y >> (8 * i)) & 255 for i in range(4))
                    from fractions import Fraction
                    vals = [float(codes.fp16_value(codes.fp16_rne(Fraction(ssum - 510) / Fraction("147.8"))))]
                else:
                    h = (s * s + s) % (1 << 32)
                    idx = (h >> (15 - p.Q)) & ((1 << p.Q) - 1)
                    word = (int(p.lut[idx, 0]) << 16) | int(p.lut[idx, 1])
                    word ^= h & (1 << 15)
                    vals = [float(codes.fp16_value(word >> 16)), float(codes.fp16_value(word & 0xFFFF))]
                for v_i, v in enumerate(vals):
                    pos = t * p.V + v_i
                    r, c = divmod(pos, 16)                    # P:833 row-major scan
                    W[I * 16 + r, J * 16 + c] = v
    return W


@pytest.mark.parametrize("code,k,V", [("3inst", 2, 1), ("1mad", 2, 1), ("hyb", 4, 2), ("hyb", 3, 2), ("3inst", 3, 1)])
def test_dense_decode_matches_scalar_definition(code, k, V):
    tiles = synth.random_tiles(32, 48, k, seed=1000 + k)
    lut = synth.gaussian_lut(9) if code == "hyb" else None
    p = gemv.Params(k=k, V=V, code=code, lut=lut)
    assert np.array_equal(gemv.dense_decode(tiles, p), _scalar_decode(tiles, p))


def test_decode_rows_matches_dense():
    tiles = synth.random_tiles(48, 32, 2, seed=3)
    p = gemv.Params()
    W = gemv.dense_decode(tiles, p)
    assert np.array_equal(gemv.decode_rows(tiles, p, [0, 17, 47]), W[[0, 17, 47]])


def test_matvec_equals_explicit_dense_product():
    m, n, B = 32, 48, 3
    tiles = synth.random_tiles(m, n, 2, seed=4)
    Wt = gemv.dense_decode(tiles, gemv.Params())
    x = synth.random_x(B, n).astype(np.float64)
    sm = synth.random_sign_bytes(m, 3001)
    sn = synth.random_sign_bytes(n, 3000)
    Hm = hadamard.hadamard(m).astype(float)
    Hn = hadamard.hadamard(n).astype(float)
    Sm = np.diag(rht.signs_from_bits(sm, m))
    Sn = np.diag(rht.signs_from_bits(sn, n))
    W = Sm @ Hm.T @ Wt @ Hn @ Sn / np.sqrt(m * n)              # W = S_m H_m^T W~ H_n S_n
    y = gemv.matvec(Wt, x, sn, sm, scale=0.7)
    assert np.allclose(y, 0.7 * x @ W.T, rtol=0, atol=1e-10)


def test_matvec_without_rht_is_plain_gemv_and_shards_concatenate():
    m, n = 64, 32
    tiles = synth.random_tiles(m, n, 2, seed=5)
    Wt = gemv.dense_decode(tiles, gemv.Params())
    x = synth.random_x(2, n).astype(np.float64)
    y = gemv.matvec(Wt, x, rht_in=False, rht_out=False, scale=2.0)
    ref = np.array([[2.0 * sum(Wt[i, j] * x[b, j] for j in range(n)) for i in range(m)] for b in range(2)])
    assert np.allclose(y, ref, rtol=1e-13, atol=1e-12)
    parts = [gemv.matvec(Wt, x, synth.random_sign_bytes(n, 1), rht_out=False, rows=(r, r + 16)) for r in range(0, m, 16)]
    full = gemv.matvec(Wt, x, synth.random_sign_bytes(n, 1), rht_out=False)
    assert np.array_equal(np.concatenate(parts, axis=1), full)
    with pytest.raises(ValueError):
        gemv.matvec(Wt, x, rows=(0, 16))


def test_single_tile_is_a_16x16_matvec():
    tiles = synth.random_tiles(16, 16, 2, seed=6)
    p = gemv.Params(code="1mad")
    Wt = gemv.dense_decode(tiles, p)
    x = synth.random_x(1, 16).astype(np.float64)
    assert np.allclose(gemv.matvec(Wt, x, rht_in=False, rht_out=False), x @ Wt.T)
