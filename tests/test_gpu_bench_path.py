"""GPU parity of exactly what bench.py runs, against the CPU oracle.

* The step's calls at the step's shapes and batch: q,k,v as ONE grouped call on 3 x (4096 x 4096),
  gate,up as one grouped call on 2 x (11008 x 4096), o (4096 x 4096) and down (4096 x 11008) as
  single calls, RHT in and out, batch 1, the auto kernel choice -- 3INST k=2 (C2) and HYB k=4 (C3).
  EVERY output row of every member is compared with the float64 oracle (relative L2 <= 1e-3,
  BASELINE.json north_star), the oracle's W~ decoded tile-row block by tile-row block.
* A bit-exact readout of each GEMV kernel's in-register / in-TMEM decode: flags = 0 (no RHT), scale 1,
  x = e_j.  x~ = binary16(e_j) is exact, so the product returns column j of the kernel's weight
  operand exactly: the binary16 weight for HYB, for 1MAD (s - 510) times fl32(5/739) (the integer
  s - 510 goes to the tensor core, 1/147.8 is folded into the fp32 scale, reading R6), for 3INST
  the exact m1 + m2 on the K-doubled mma.sync kernels (impls 3-6, reading R10) and binary16 RNE of
  m1 + m2 -- qtip_decode's value -- on the tcgen05 kernel (impl 7).  Columns cover both K halves
  of a 16-column tile, the last tile column (windows that wrap past the tile's last stream bit),
  several cells and the last column.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import codes, gemv, rht, trellis

pytestmark = pytest.mark.gpu

TOL = 1e-3


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def oracle_matvec_blocked(tiles, p, x, sign_n, sign_m, scale, rows_per_block=1024):
    """gemv.matvec computed with W~ decoded one block of tile rows at a time (same arithmetic:
    float64 x~ = RHT(x), y~ = x~ W~^T, y = RHT^-1(y~) * scale), bounded memory at 11008 x 4096."""
    m, n = tiles.shape[0] * 16, tiles.shape[1] * 16
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    xt = rht.rht_forward(x, sign_n, n)
    yt = np.zeros((x.shape[0], m))
    tr = rows_per_block // 16
    for I0 in range(0, tiles.shape[0], tr):
        W = gemv.dense_decode(tiles[I0:I0 + tr], p)
        yt[:, 16 * I0:16 * I0 + W.shape[0]] = xt @ W.T
    return scale * rht.rht_inverse(yt, sign_m, m)


def _layers(cuda_lib, code, k, m, n, G, seed0):
    from paper_2406_11235_b200.layer import QTIPLinear
    lut = synth.gaussian_lut(9) if code == "hyb" else None
    out = []
    for g in range(G):
        tiles = synth.random_tiles(m, n, k, seed=seed0 + g)
        sm, sn = synth.random_sign_bytes(m, 3001 + seed0 + g), synth.random_sign_bytes(n, 3000 + seed0 + g)
        lay = QTIPLinear(m, n, code=code, k=k).load_tiles(tiles, sm, sn, scale=1.0, lut=lut)
        out.append((lay, tiles, sm, sn))
    return out, lut


@pytest.mark.parametrize("code,k", [("3inst", 2), ("hyb", 4)])
@pytest.mark.parametrize("what,m,n,G", [("qkv", 4096, 4096, 3), ("o", 4096, 4096, 1), ("gate_up", 11008, 4096, 2),
                                        ("down", 4096, 11008, 1)])
def test_bench_step_calls_every_row_vs_oracle(cuda_lib, code, k, what, m, n, G):
    from paper_2406_11235_b200.layer import forward_group
    layers, lut = _layers(cuda_lib, code, k, m, n, G, seed0=1000 + 10 * G + (m != n))
    x = synth.random_x(1, n, seed=2000 + n)
    dx = torch.from_numpy(x).cuda()
    if G > 1:
        ys = [y.cpu().numpy() for y in forward_group([l for l, *_ in layers], dx)]   # the bench's grouped call
    else:
        ys = [layers[0][0](dx).cpu().numpy()]
    p = gemv.Params(k=k, V=2 if code == "hyb" else 1, code=code, lut=lut)
    for (lay, tiles, sm, sn), y in zip(layers, ys):
        ref = oracle_matvec_blocked(tiles, p, x, sn, sm, 1.0)
        assert y.shape == ref.shape
        assert rel_l2(y, ref) <= TOL


@pytest.mark.parametrize("code,k,B", [("hyb", 4, 16), ("hyb", 4, 64), ("3inst", 2, 64)])
def test_batched_tcgen05_slab_ring_wraps_vs_oracle(cuda_lib, code, k, B):
    """The stream-K tcgen05 kernel (impl 7) at batch 16 / 64 on a 4096 x 8192 layer: 2048 cells over
    the SMs is ~14 per CTA, more than the x~ slab slots that fit next to the HYB LUT at B = 16 (11) or
    at B = 64 (2 with the LUT, 10 without), so every slot is refilled while the ring runs; every row
    of every batch column vs the float64 oracle."""
    from paper_2406_11235_b200 import qtip
    m, n = 4096, 8192
    layers, lut = _layers(cuda_lib, code, k, m, n, 1, seed0=1700 + B)
    lay, tiles, sm, sn = layers[0]
    x = synth.random_x(B, n, seed=2100 + B)
    qtip.set_matvec_impl(7)
    try:
        y = lay(torch.from_numpy(x).cuda()).cpu().numpy()
    finally:
        qtip.set_matvec_impl(0)
    p = gemv.Params(k=k, V=2 if code == "hyb" else 1, code=code, lut=lut)
    ref = oracle_matvec_blocked(tiles, p, x, sn, sm, 1.0)
    assert y.shape == ref.shape
    for b in range(B):
        assert rel_l2(y[b], ref[b]) <= TOL, b


def _tile_positions(m, n, j):
    """(I, J, r, c) of the weights W~[:, j] and their sequence positions p = 16 r + c."""
    rows = np.arange(m)
    return rows // 16, j // 16, rows % 16, j % 16


def _expected_column(tiles, code, k, lut, j, impl):
    """Column j of the GEMV's weight operand times e_j, from the oracle's integers."""
    m = tiles.shape[0] * 16
    I, J, r, c = _tile_positions(m, tiles.shape[1] * 16, j)
    V = 2 if code == "hyb" else 1
    st = trellis.tile_states(tiles[:, J], 16, k, V, 256)                     # (m/16, 256/V) states of column tile J
    if code == "hyb":
        t = (16 * r + c) // 2
        pair = codes.decode_hyb(st[I, t].astype(np.uint64), lut, 9)          # (m, 2) binary16 (c0, c1)
        bits = pair[np.arange(m), c % 2]
        return codes.f16_to_f64(bits).astype(np.float32)
    x = st[I, 16 * r + c].astype(np.uint64)
    if code == "1mad":
        s = codes.byte_sum(codes.lcg(x, codes.A_1MAD, codes.B_1MAD))
        return (np.float32(1.0) * (s - 510).astype(np.float32) * np.float32(5.0 / 739.0)).astype(np.float32)
    m1, m2 = codes.inst3_halves(x)
    if impl == 7:                                                          # binary16 RNE(m1 + m2)
        return codes.f16_to_f64(codes.decode_3inst(x)).astype(np.float32)
    return (codes.f16_to_f64(m1) + codes.f16_to_f64(m2)).astype(np.float32)  # exact, K-doubled


@pytest.mark.parametrize("impl", [3, 4, 5, 6, 7])
@pytest.mark.parametrize("code,k", [("3inst", 2), ("1mad", 2), ("hyb", 4), ("hyb", 3), ("3inst", 3)])
def test_gemv_weight_operand_readout_is_bit_exact(cuda_lib, impl, code, k):
    from paper_2406_11235_b200.layer import QTIPLinear
    m, n = 384, 768                                                        # 3 row blocks x 6 cells
    lut = synth.gaussian_lut(9) if code == "hyb" else None
    tiles = synth.random_tiles(m, n, k, seed=700 + k)
    lay = QTIPLinear(m, n, code=code, k=k).load_tiles(tiles, synth.random_sign_bytes(m, 1),
                                                       synth.random_sign_bytes(n, 2), scale=1.0, lut=lut)
    cols = [0, 1, 7, 8, 9, 14, 15, 16, 127, 128, 255, 300, 511, 640, 767]
    X = np.zeros((len(cols), n), dtype=np.float32)
    for b, j in enumerate(cols):
        X[b, j] = 1.0
    cuda_lib.set_matvec_impl(impl)
    try:
        ys = []
        for b0 in range(0, len(cols), 4):                                  # batch <= 4 on every kernel
            xb = torch.from_numpy(X[b0:b0 + 4]).cuda()
            ys.append(lay(xb, flags=0).cpu().numpy())
        Y = np.concatenate(ys, axis=0)
    finally:
        cuda_lib.set_matvec_impl(0)
    for b, j in enumerate(cols):
        want = _expected_column(tiles, code, k, lut, j, impl)
        got = Y[b].astype(np.float32)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (impl, code, k, j)
