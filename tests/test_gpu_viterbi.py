"""GPU tail-biting quantizer (qtip_viterbi_tailbite, Algorithm 4) vs the CPU oracle's binary32 DP
on identical seeded inputs: walks and costs bit-exact (the argmins are taken in binary32 on both
sides, reading R17), and the walks pack into a valid tail-biting stream that decodes to the
quantized weights."""
import numpy as np
import pytest
import torch

import synth
from oracle import codes, viterbi

pytestmark = pytest.mark.gpu


def _src(code, nseq, T, seed):
    tab = codes.code_table(code, 16)
    S = synth.gaussian_source(nseq, T, seed=seed)
    return (S.astype(np.float32) * np.float32(tab.std())).astype(np.float32), tab.astype(np.float32)


@pytest.mark.parametrize("code,k,nseq,T", [("3inst", 2, 64, 256), ("1mad", 2, 40, 256), ("3inst", 3, 24, 128),
                                           ("1mad", 3, 9, 256), ("3inst", 2, 300, 64), ("3inst", 2, 3, 2),
                                           ("3inst", 4, 6, 256), ("1mad", 4, 4, 128), ("3inst", 4, 5, 2),
                                           ("1mad", 4, 3, 16)])
def test_viterbi_matches_oracle_bit_exact(cuda_lib, code, k, nseq, T):
    from paper_2406_11235_b200.quantize import QTIPQuantizer
    src, tab = _src(code, nseq, T, seed=5000 + T + k)
    st, cost = QTIPQuantizer(code, k).encode(torch.from_numpy(src).cuda())
    ref_st, ref_cost = viterbi.tailbite_encode_f32_batch(src, 16, k, 1, tab)
    assert np.array_equal(st.cpu().numpy().view(np.uint32), ref_st)
    assert np.array_equal(cost.cpu().numpy(), ref_cost)


def test_c1_quantize_pack_decode_roundtrip(cuda_lib):
    """Config C1 end to end on the GPU: 256 x 256 3INST k=2 tiles of i.i.d. N(0,1) ->
    Algorithm 4 walks -> qtip_pack_states (rejects non-tail-biting walks) -> qtip_decode; the
    decoded weights reproduce each tile's reported squared error and sit near Table 1's MSE."""
    from paper_2406_11235_b200 import qtip
    from paper_2406_11235_b200.layer import QTIPLinear
    from paper_2406_11235_b200.quantize import QTIPQuantizer
    m = n = 256
    tab = codes.code_table("3inst", 16)
    sd = np.float32(tab.std())
    W = synth.gaussian_source(m, n, seed=5000).astype(np.float32)            # RHT-domain weights ~ N(0,1)
    q = QTIPQuantizer("3inst", 2)
    walks, cost = q.quantize_tiles(torch.from_numpy(W), sd)
    layer = QTIPLinear(m, n, code="3inst", k=2)
    qtip.qtip_pack_states(layer.p, m, n, walks, layer.packed)
    dec = layer.decode(out_f32=True).cpu().numpy()                           # raw code values
    err = (dec - W * sd).reshape(m // 16, 16, n // 16, 16).transpose(0, 2, 1, 3).reshape(-1, 256)
    c = cost.cpu().numpy()
    np.testing.assert_allclose((err.astype(np.float64) ** 2).sum(axis=1), c, rtol=1e-4)
    mse = float(((dec / sd - W) ** 2).mean())
    assert 0.060 < mse < 0.080                                                # Table 1, 3INST tail-biting ~0.068


@pytest.mark.parametrize("k,nseq,T", [(2, 8, 256), (3, 6, 128), (4, 4, 32), (2, 130, 16), (4, 3, 2)])
def test_viterbi_hyb_matches_oracle_bit_exact(cuda_lib, k, nseq, T):
    """HYB (V = 2) through the GPU quantizer: 2^(2k) predecessors per group, LUT code
    with the bit-15 sign, walks and costs bit-exact vs the oracle's binary32 Algorithm 4."""
    from paper_2406_11235_b200.quantize import QTIPQuantizer
    lut = synth.gaussian_lut(9, 4000)
    tab = codes.code_table("hyb", 16, lut=lut, Q=9)
    S = synth.gaussian_source(nseq, T, seed=6000 + k + T)
    src = (S.astype(np.float32) * np.float32(tab.std())).astype(np.float32)
    st, cost = QTIPQuantizer("hyb", k, lut=lut).encode(torch.from_numpy(src).cuda())
    ref_st, ref_cost = viterbi.tailbite_encode_f32_batch(src, 16, k, 2, tab.astype(np.float32))
    assert np.array_equal(st.cpu().numpy().view(np.uint32), ref_st)
    assert np.array_equal(cost.cpu().numpy(), ref_cost)


def test_hyb_quantize_pack_decode_roundtrip(cuda_lib):
    """HYB k=2 tiles -> GPU walks -> pack -> decode reproduces the reported squared errors."""
    from paper_2406_11235_b200 import qtip
    from paper_2406_11235_b200.layer import QTIPLinear
    from paper_2406_11235_b200.quantize import QTIPQuantizer
    m, n, k = 64, 128, 2
    lut = synth.gaussian_lut(9, 4000)
    tab = codes.code_table("hyb", 16, lut=lut, Q=9)
    sd = np.float32(tab.std())
    W = synth.gaussian_source(m, n, seed=6100).astype(np.float32)
    walks, cost = QTIPQuantizer("hyb", k, lut=lut).quantize_tiles(torch.from_numpy(W), sd)
    layer = QTIPLinear(m, n, code="hyb", k=k)
    layer.load_tiles(synth.random_tiles(m, n, k, seed=1), synth.random_sign_bytes(m, 1), synth.random_sign_bytes(n, 2),
                     lut=lut)
    qtip.qtip_pack_states(layer.p, m, n, walks, layer.packed)
    dec = layer.decode(out_f32=True).cpu().numpy()
    err = (dec - W * sd).reshape(m // 16, 16, n // 16, 16).transpose(0, 2, 1, 3).reshape(-1, 256)
    np.testing.assert_allclose((err.astype(np.float64) ** 2).sum(axis=1), cost.cpu().numpy(), rtol=1e-4)


def test_no_sequences_is_a_no_op(cuda_lib):
    """nseq = 0: empty walks and costs, no launch (the ABI itself refuses nseq < 1)."""
    import torch
    from paper_2406_11235_b200.quantize import QTIPQuantizer
    q = QTIPQuantizer("3inst", 2)
    c0 = cuda_lib.launch_count()
    w, c = q.encode(torch.empty((0, 256), dtype=torch.float32, device="cuda"))
    assert tuple(w.shape) == (0, 256) and tuple(c.shape) == (0,) and cuda_lib.launch_count() == c0


@pytest.mark.parametrize("code,k", [("3inst", 2), ("1mad", 4)])
def test_quantize_matrix_scan_and_scale_bit_exact(cuda_lib, code, k):
    """qtip_quantize_matrix does the block scan (16 x 16 tiles, row-major) and the scaling into
    code units (R9) in the library: its walks and costs equal the oracle's binary32 Algorithm 4 on the
    sequences cut and scaled on the host."""
    from paper_2406_11235_b200.quantize import QTIPQuantizer
    m, n = 64, 48
    tab = codes.code_table(code, 16)
    sd = np.float32(tab.std())
    W = synth.gaussian_source(m, n, seed=5100 + k).astype(np.float32)
    walks, cost = QTIPQuantizer(code, k).quantize_tiles(torch.from_numpy(W), sd)
    seqs = (W.reshape(m // 16, 16, n // 16, 16).transpose(0, 2, 1, 3).reshape(-1, 256) * sd).astype(np.float32)
    ref_st, ref_cost = viterbi.tailbite_encode_f32_batch(seqs, 16, k, 1, tab.astype(np.float32))
    assert np.array_equal(walks.reshape(-1, 256), ref_st)
    assert np.array_equal(cost.cpu().numpy(), ref_cost)
