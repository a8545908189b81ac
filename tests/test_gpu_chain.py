"""GPU parity of the chain kernel (impl 8: qtip_chain_run, k_chain.cu) against the CPU oracle.

A chain applies its layers in stages; stage 0 reads the external x, every later stage reads the
output y of one layer of the previous stage (a decode step: q, k, v -> o -> gate, up -> down -> next
q, k, v).  Each layer's y is compared, every row, with the float64 oracle (gemv.matvec: RHT in,
decoded W~, RHT out) applied to that layer's actual input -- x for stage 0, the
GPU's own y_src otherwise -- at relative L2 <= 1e-3 (BASELINE.json north_star), so the bar does not
compound along the chain.  Shapes cover power-of-two and Paley (28, 344) Hadamard sides on both
the forward (n) and inverse (m) transforms, stages of 1-4 layers, batches 1-16, tiny stages with
fewer cells than SMs (empty ranges), and the full 7B block (3 x 4096^2, 4096^2, 2 x 11008 x 4096,
4096 x 11008) followed by the next block's q, k, v.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import gemv

from test_gpu_bench_path import oracle_matvec_blocked, rel_l2

pytestmark = pytest.mark.gpu
TOL = 1e-3
VAR = {"3inst": 1.547, "1mad": 1.0, "hyb": 1.0}


def build(code, k, stages, B, seed=0):
    """stages: list of ([(m, n), ...], src).  Returns the QTIPChain and per-stage (tiles, sm, sn, scale)."""
    from paper_2406_11235_b200.layer import QTIPChain, QTIPLinear
    lut = synth.gaussian_lut(9) if code == "hyb" else None
    spec, info = [], []
    for si, (shapes, src) in enumerate(stages):
        lays, inf = [], []
        for li, (m, n) in enumerate(shapes):
            s0 = seed + 100 * si + li
            tiles = synth.random_tiles(m, n, k, seed=1000 + s0)
            sm, sn = synth.random_sign_bytes(m, 3001 + s0), synth.random_sign_bytes(n, 3000 + s0)
            scale = 1.0 / np.sqrt(n * VAR[code])
            lays.append(QTIPLinear(m, n, code=code, k=k).load_tiles(tiles, sm, sn, scale=scale, lut=lut))
            inf.append((tiles, sm, sn, scale))
        spec.append((lays, src))
        info.append(inf)
    return QTIPChain(spec, B=B), info, lut


def check(chain, info, lut, code, k, stages, x):
    p = gemv.Params(k=k, V=2 if code == "hyb" else 1, code=code, lut=lut)
    outs = [[y.cpu().numpy() for y in st] for st in chain.outs]
    worst = 0.0
    for si, (shapes, src) in enumerate(stages):
        xin = x if si == 0 else outs[si - 1][src]
        for li, (tiles, sm, sn, scale) in enumerate(info[si]):
            ref = oracle_matvec_blocked(tiles, p, xin, sn, sm, scale)
            err = rel_l2(outs[si][li], ref)
            worst = max(worst, err)
            assert err <= TOL, (si, li, shapes[li], err)
    return worst


SMALL = [([(512, 256), (512, 256)], 0), ([(256, 512)], 1), ([(448, 256), (448, 256), (448, 256)], 0),
         ([(256, 448)], 0), ([(11008, 256)], 0), ([(256, 11008)], 0)]


@pytest.mark.parametrize("code,k", [("3inst", 2), ("1mad", 2), ("hyb", 4), ("hyb", 3), ("3inst", 3), ("1mad", 4),
                                    ("hyb", 2)])
def test_chain_small_every_layer_vs_oracle(cuda_lib, code, k):
    chain, info, lut = build(code, k, SMALL, B=1)
    x = synth.random_x(1, 256, seed=2000)
    chain(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    check(chain, info, lut, code, k, SMALL, x)


@pytest.mark.parametrize("B", [2, 3, 4, 8, 16])
@pytest.mark.parametrize("code,k", [("3inst", 2), ("hyb", 4)])
def test_chain_batches_vs_oracle(cuda_lib, code, k, B):
    st = SMALL[:4]
    chain, info, lut = build(code, k, st, B=B, seed=7)
    x = synth.random_x(B, 256, seed=2100 + B)
    chain(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    check(chain, info, lut, code, k, st, x)


def test_chain_tiny_stages_and_repeat_bitwise(cuda_lib):
    # stages of 1-2 cells (most CTAs have empty ranges), a 4-layer stage, odd Hadamard sides
    st = [([(128, 128)], 0), ([(224, 128), (224, 128), (224, 128), (224, 128)], 0), ([(16, 224)], 3),
          ([(192, 16)], 0), ([(128, 192)], 0)]
    chain, info, lut = build("3inst", 2, st, B=1, seed=11)
    x = torch.from_numpy(synth.random_x(1, 128, seed=2200)).cuda()
    chain(x)
    first = [[y.clone() for y in s] for s in chain.outs]
    check(chain, info, lut, "3inst", 2, st, x.cpu().numpy())
    for _ in range(3):
        chain(x)
    torch.cuda.synchronize()
    for a, b in zip(first, chain.outs):
        for u, v in zip(a, b):
            assert torch.equal(u, v)


@pytest.mark.parametrize("code,k", [("3inst", 2), ("hyb", 4)])
def test_chain_7b_block_every_row_vs_oracle(cuda_lib, code, k):
    st = [([(4096, 4096)] * 3, 0), ([(4096, 4096)], 2), ([(11008, 4096)] * 2, 0), ([(4096, 11008)], 0),
          ([(4096, 4096)] * 3, 0)]
    chain, info, lut = build(code, k, st, B=1, seed=20)
    x = synth.random_x(1, 4096, seed=2300)
    chain(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    check(chain, info, lut, code, k, st, x)


def test_chain_matches_per_layer_calls(cuda_lib):
    """The same chain through per-layer QTIPLinear calls (RHT kernels + GEMV) agrees to fp32 rounding."""
    st = SMALL[:4]
    chain, info, lut = build("hyb", 4, st, B=2, seed=5)
    x = torch.from_numpy(synth.random_x(2, 256, seed=2400)).cuda()
    chain(x)
    idx = 0
    outs = []
    for si, (shapes, src) in enumerate(st):
        xin = x if si == 0 else outs[si - 1][src]
        cur = []
        for li in range(len(shapes)):
            cur.append(chain.layers[idx](xin))
            idx += 1
        outs.append(cur)
    for a, b in zip(chain.outs, outs):
        for u, v in zip(a, b):
            assert rel_l2(u.cpu().numpy(), v.cpu().numpy()) <= 2e-3
