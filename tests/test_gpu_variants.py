"""GPU parity of the NEXT-3 code variants (k_variant.cu) against the CPU oracle: the lookup-only code
(QTIP_CODE_LUT: L = 14, V = 1, T_x x T_y = 32 x 8; also 16 x 16 and other L) and HYB
with a 1-D codebook (V = 1, Q = 6).  Decode bit-exact; matvec relative L2 <= 1e-3
(BASELINE.json north_star) for every row, RHT in/out, several k, batches and shapes incl. Paley sides
and a row range."""
import ctypes

import numpy as np
import pytest
import torch

import synth
from oracle import gemv

from test_gpu_bench_path import rel_l2

pytestmark = pytest.mark.gpu


def _layer(cuda_lib, code, k, m, n, seed, L=None, Tx=None):
    from paper_2406_11235_b200.layer import QTIPLinear
    lay = QTIPLinear(m, n, code=code, k=k)
    if L is not None:
        lay.p.L = L
    if Tx is not None:
        lay.p.Tx, lay.p.Ty = Tx, 256 // Tx
    Tx_, Ty_ = lay.p.Tx, lay.p.Ty
    tiles = synth.random_tiles(m, n, k, seed=seed, Tx=Tx_, Ty=Ty_)
    lut = synth.gaussian_table(lay.p.L if code == "lut" else lay.p.Q, seed=4001 + seed)
    sm, sn = synth.random_sign_bytes(m, 3001 + seed), synth.random_sign_bytes(n, 3000 + seed)
    lay.load_tiles(tiles, sm, sn, scale=0.3, lut=lut)
    p = gemv.Params(L=lay.p.L, k=k, V=1, code=code, Q=lay.p.Q, lut=lut, Tx=Tx_, Ty=Ty_)
    return lay, tiles, lut, sm, sn, p


CASES = [("lut", 2, None, None), ("lut", 3, None, None), ("lut", 4, None, None), ("lut", 2, 16, 16), ("lut", 2, 12, 32),
         ("hyb1", 2, None, None), ("hyb1", 3, None, None), ("hyb1", 4, None, None)]


@pytest.mark.parametrize("code,k,L,Tx", CASES)
def test_variant_decode_bit_exact(cuda_lib, code, k, L, Tx):
    lay, tiles, lut, sm, sn, p = _layer(cuda_lib, code, k, 384, 256, seed=31 + k, L=L, Tx=Tx)
    got = lay.decode().cpu().numpy().view(np.uint16)
    want = gemv.dense_decode(tiles, p).astype(np.float16).view(np.uint16)
    assert np.array_equal(got, want)
    got32 = lay.decode(out_f32=True).cpu().numpy()
    assert np.array_equal(got32, gemv.dense_decode(tiles, p).astype(np.float32))


@pytest.mark.parametrize("B", [1, 4, 16])
@pytest.mark.parametrize("code,k,L,Tx", CASES)
@pytest.mark.parametrize("m,n", [(256, 512), (448, 224), (1024, 4096)])
def test_variant_matvec_vs_oracle(cuda_lib, code, k, L, Tx, B, m, n):
    lay, tiles, lut, sm, sn, p = _layer(cuda_lib, code, k, m, n, seed=41 + k + B, L=L, Tx=Tx)
    x = synth.random_x(B, n, seed=2000 + B)
    y = lay(torch.from_numpy(x).cuda()).cpu().numpy()
    ref = gemv.matvec(gemv.dense_decode(tiles, p), x, sn, sm, scale=0.3)
    assert rel_l2(y, ref) <= 1e-3


def test_variant_row_range_and_no_rht(cuda_lib):
    from paper_2406_11235_b200 import qtip
    lay, tiles, lut, sm, sn, p = _layer(cuda_lib, "lut", 2, 512, 256, seed=5)
    x = synth.random_x(2, 256, seed=7)
    y = lay(torch.from_numpy(x).cuda(), flags=qtip.QTIP_RHT_IN, rows=(128, 384)).cpu().numpy()
    ref = gemv.matvec(gemv.dense_decode(tiles, p), x, sn, sm, scale=0.3, rht_out=False, rows=(128, 384))
    assert rel_l2(y, ref) <= 1e-3
    y0 = lay(torch.from_numpy(x).cuda(), flags=0).cpu().numpy()
    ref0 = gemv.matvec(gemv.dense_decode(tiles, p), x, None, None, scale=0.3, rht_in=False, rht_out=False)
    assert rel_l2(y0, ref0) <= 1e-6                          # float32 x~, exact binary16 weights


def test_variant_lut_7b_layer_vs_oracle(cuda_lib):
    """The paper's setting (L = 14, 32 x 8) at a Llama-2-7B shape, every row."""
    lay, tiles, lut, sm, sn, p = _layer(cuda_lib, "lut", 2, 4096, 4096, seed=3)
    x = synth.random_x(1, 4096, seed=2001)
    y = lay(torch.from_numpy(x).cuda()).cpu().numpy()
    ref = gemv.matvec(gemv.dense_decode(tiles, p), x, sn, sm, scale=0.3)
    assert rel_l2(y, ref) <= 1e-3
