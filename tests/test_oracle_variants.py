"""Pins of the oracle's code variants: HYB with a 1-D codebook (Q = 6, V = 1,
PAPER.md:607-609) and the lookup-only code (L = 14, V = 1, T_x = 32, T_y = 8)."""
import numpy as np

import synth
from oracle import codes, gemv, trellis


def test_hyb1_is_the_flipped_element_of_the_2d_code():
    # P:317 flips bit 15 of the LUT word; with V = 2 that is the sign of the second element, so a 1-D
    # codebook equal to the second column reproduces it exactly, for every 16-bit state
    lut2 = synth.gaussian_lut(6, seed=7)
    xs = np.arange(1 << 16, dtype=np.uint64)
    v2 = codes.decode_hyb(xs, lut2, 6)
    v1 = codes.decode_hyb1(xs, lut2[:, 1], 6)
    assert np.array_equal(v1, v2[:, 1])


def test_hyb1_index_and_sign_counts_q6():
    # over all 2^16 states each of the 2^6 indices is hit exactly 2^10 times, each with both signs
    # equally often (the Q = 9 analogue of SURVEY Appendix A: 128 hits per index)
    xs = np.arange(1 << 16, dtype=np.uint64)
    h = codes.hyb_hash(xs)
    idx = codes.hyb_index(h, 6)
    assert np.array_equal(np.bincount(idx, minlength=64), np.full(64, 1024))
    sign = ((h >> np.uint64(15)) & np.uint64(1)).astype(np.int64)
    assert np.bincount(idx * 2 + sign, minlength=128).min() > 0
    # golden: x = 3 -> h = 12 -> idx 0, bit 15 clear; x = 0xFFFF -> h = 0xFFFF0000 -> idx 0
    assert int(codes.hyb_index(codes.hyb_hash(np.uint64(3)), 6)) == 0
    lut1 = np.arange(64, dtype=np.uint16) + 0x3C00           # 1.0, 1.0009765625, ...
    assert int(codes.decode_hyb1(np.uint64(3), lut1, 6)) == 0x3C00
    assert int(codes.decode_hyb1(np.uint64(0xFFFF), lut1, 6)) == 0x3C00       # bit 15 of 0xFFFF0000 is 0
    x = np.uint64(0x1234)                                     # h = 0x014B6CC4: bit 15 clear
    assert int(codes.decode_hyb1(x, lut1, 6)) == 0x3C00 + ((0x014B6CC4 >> 9) & 63)


def test_lut_code_reads_the_state_table():
    # the identity table (binary16 bit pattern x for state x: distinct finite values) makes the
    # decoded weights the states themselves
    L, k = 14, 2
    lut = np.arange(1 << L, dtype=np.uint16)
    assert np.array_equal(codes.decode_lut(np.arange(1 << L), lut), lut)
    rng = np.random.default_rng(3)
    # a random closed walk of the (14, 2, 1) trellis, packed tail-biting into 512 bits
    bits = rng.integers(0, 2, 512)
    states = [trellis.window(bits, t, L, k, 1, True) for t in range(256)]
    for t in range(255):                                      # edge rule
        assert trellis.is_edge(states[t], states[t + 1], L, k, 1)
    tile = np.packbits(bits.astype(np.uint8), bitorder="big")[None, None, :]
    p = gemv.Params(L=L, k=k, V=1, code="lut", lut=lut, Tx=32, Ty=8)
    W = gemv.dense_decode(tile, p)
    assert W.shape == (32, 8)
    # row-major scan of the 32 x 8 block (P:833 with T_x = 32, T_y = 8): position p = 8 r + c
    assert np.array_equal(W.reshape(-1), codes.f16_to_f64(np.array(states, dtype=np.uint16)))


def test_lut_code_tiles_layout_32x8():
    m, n, k = 64, 32, 2
    tiles = synth.random_tiles(m, n, k, seed=9, Tx=32, Ty=8)
    assert tiles.shape == (2, 4, 64)
    lut = synth.gaussian_table(14)
    p = gemv.Params(L=14, k=k, V=1, code="lut", lut=lut, Tx=32, Ty=8)
    W = gemv.dense_decode(tiles, p)
    for I in range(2):
        for J in range(4):
            st = trellis.tile_states(tiles[I, J], 14, k, 1, 256)
            vals = codes.f16_to_f64(lut[st])
            assert np.array_equal(W[32 * I:32 * I + 32, 8 * J:8 * J + 8].reshape(-1), vals)


def test_lut_code_quantizes_a_gaussian_near_the_rate_bound():
    """The lookup-only code is a trellis code like the others: Algorithm 4 with a 2^14 N(0,1) table
    reaches Table 1's regime at k = 2 (tail-biting MSE ~0.068-0.07 for L = 16 codes; L = 14 is a
    little worse but far below the scalar-quantizer 0.1175 and above D_R = 0.0625)."""
    from oracle import viterbi
    L, k = 14, 2
    tab = codes.f16_to_f64(synth.gaussian_table(L)).astype(np.float64)
    tab = tab / tab.std()
    src = synth.gaussian_source(8, 256, seed=5003)
    st, _ = viterbi.tailbite_encode_batch(src, L, k, 1, tab)
    mse = float(np.mean((tab[np.asarray(st)] - src) ** 2))
    assert codes.distortion_rate_bound(k) < mse < 0.085, mse
