"""GPU BlockLDLQ (Algorithm 5) against the oracle's Algorithm 5.

The GPU driver (QTIPQuantizer.blockldlq) rounds every T_x x T_y = 16 x 16 sequence with the library's
Algorithm 4 (binary32 DP) and reconstructs with the library's decoder; the factorisation and the
feedback product are fp32/fp64 library linear algebra.  The oracle runs the same algorithm in float64
with its binary32 Algorithm 4 as the rounding step (`quantize=`), so:
  * the rightmost block column has no feedback (x = W): its walks are bit-exact;
  * H = I has no feedback anywhere: the whole result equals blockwise Algorithm 4 (bit-exact);
  * elsewhere x differs from the oracle's only by fp32 rounding of the feedback, so near-tied
    argmins may differ: the walks agree almost everywhere and the proxy loss matches closely and
    beats rounding without feedback.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import codes, ldlq, viterbi

pytestmark = pytest.mark.gpu

K = 2


def _setup(m, n, seed, code="3inst"):
    lut = synth.gaussian_lut(9, 4000) if code == "hyb" else None
    tab = codes.code_table(code, 16, lut=lut, Q=9) if code == "hyb" else codes.code_table(code, 16)
    sd = np.float32(tab.std())
    W = synth.gaussian_source(m, n, seed=seed).astype(np.float32)
    return tab, sd, W, lut


def _oracle(W, H, tab, sd, V=1):
    quant = lambda S: viterbi.tailbite_encode_f32_batch((S * np.float64(sd)).astype(np.float32), 16, K, V,  # noqa: E731
                                                        tab.astype(np.float32))
    return ldlq.blockldlq(W.astype(np.float64), H, 16, 16, 16, K, V, tab / np.float64(sd), quantize=quant)


def test_blockldlq_identity_hessian_is_blockwise_algorithm4(cuda_lib):
    from paper_2406_11235_b200.quantize import QTIPQuantizer
    m, n = 64, 48
    tab, sd, W, _ = _setup(m, n, 7100)
    q = QTIPQuantizer("3inst", K)
    What, walks = q.blockldlq(torch.from_numpy(W), np.eye(n), float(sd))
    ref_walks, _ = q.quantize_tiles(torch.from_numpy(W), sd)                 # [m/16][n/16][256]
    assert np.array_equal(walks.transpose(1, 0, 2), ref_walks)
    ref = (tab[ref_walks.reshape(m // 16, n // 16, 16, 16).transpose(0, 2, 1, 3).reshape(m, n)] / np.float64(sd))
    assert np.allclose(What.cpu().numpy(), ref, rtol=1e-6, atol=0)


@pytest.mark.parametrize("code", ["3inst", "hyb"])
def test_blockldlq_matches_oracle_algorithm5(cuda_lib, code):
    from paper_2406_11235_b200.quantize import QTIPQuantizer
    m, n = 48, 64
    tab, sd, W, lut = _setup(m, n, 7200, code)
    V = 2 if code == "hyb" else 1
    H = synth.synthetic_hessian(n, rho=0.9, seed=7201)
    q = QTIPQuantizer(code, K, lut=lut)
    What, walks = q.blockldlq(torch.from_numpy(W), H, float(sd))
    Wo, walks_o = _oracle(W, H, tab, sd, V)
    assert np.array_equal(walks[-1], walks_o[-1])                           # no feedback: bit-exact
    agree = np.mean(walks == walks_o)
    assert agree > 0.9, agree
    Wg = What.cpu().numpy().astype(np.float64)
    loss_g, loss_o = ldlq.proxy_loss(W, Wg, H), ldlq.proxy_loss(W, Wo, H)
    assert abs(loss_g - loss_o) <= 0.02 * loss_o, (loss_g, loss_o)
    # the feedback helps: rounding every block on its own (H = I) is worse under H
    Wi, _ = q.blockldlq(torch.from_numpy(W), np.eye(n), float(sd))
    assert loss_g < ldlq.proxy_loss(W, Wi.cpu().numpy().astype(np.float64), H)
