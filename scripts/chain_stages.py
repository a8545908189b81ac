#!/usr/bin/env python
"""Stage-by-stage check of one small chain: the plan's x~ (RHT-in) against the oracle's RHT, its y~
against W~ x~ computed by the oracle from the GPU's x~, and y against the oracle's inverse RHT of the
GPU's y~ -- locates which part of the chain kernel disagrees.

usage: python scripts/chain_stages.py [code] [k] [B]
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2406_11235_b200 import qtip  # noqa: E402
from oracle import gemv, rht  # noqa: E402
import test_gpu_chain as T  # noqa: E402

code = sys.argv[1] if len(sys.argv) > 1 else "3inst"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
lib = qtip.load()
fn = lib.qtip_internal_chain_buffers
fn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p)]
stages = T.SMALL
chain, info, lut = T.build(code, k, stages, B=B)
x = np.random.default_rng(0).standard_normal((B, 256)).astype(np.float32)
chain(torch.from_numpy(x).cuda())
torch.cuda.synchronize()
p = gemv.Params(k=k, V=2 if code == "hyb" else 1, code=code, lut=lut)
BP = 1 if B <= 1 else 2 if B <= 2 else 4 if B <= 4 else 8 if B <= 8 else 16
li = 0
outs = [[y.cpu().numpy() for y in st] for st in chain.outs]


for si, (shapes, src) in enumerate(stages):
    xin = x if si == 0 else outs[si - 1][src]
    for j, (tiles, sm, sn, scale) in enumerate(info[si]):
        m, n = shapes[j]
        xt_p, yt_p = ctypes.c_void_p(), ctypes.c_void_p()
        assert fn(chain._plan, li, ctypes.byref(xt_p), ctypes.byref(yt_p)) == 0
        npad = (n + 127) // 128 * 128
        mpad = (m + 127) // 128 * 128
        xt_t = torch.empty(npad * BP, dtype=torch.float16, device="cuda")
        yt_t = torch.empty(B * mpad, dtype=torch.float32, device="cuda")
        torch.cuda.synchronize()
        cp = lib.qtip_internal_copy
        cp.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]
        cp.restype = ctypes.c_int
        assert cp(ctypes.c_void_p(xt_t.data_ptr()), xt_p, npad * BP * 2) == 0
        assert cp(ctypes.c_void_p(yt_t.data_ptr()), yt_p, B * mpad * 4) == 0
        xt_g = xt_t.cpu().numpy().astype(np.float64).reshape(npad // 8, BP, 8).transpose(1, 0, 2).reshape(BP, npad)[:B, :n]
        yt_g = yt_t.cpu().numpy().astype(np.float64).reshape(B, mpad)[:, :m]
        xt_ref = rht.rht_forward(np.atleast_2d(xin).astype(np.float64), sn, n)
        e_xt = np.linalg.norm(xt_g - xt_ref) / np.linalg.norm(xt_ref)
        W = gemv.dense_decode(tiles, p)
        yt_ref = xt_g @ W.T
        e_yt = np.linalg.norm(yt_g - yt_ref) / np.linalg.norm(yt_ref)
        y_ref = scale * rht.rht_inverse(yt_g, sm, m)
        e_y = np.linalg.norm(outs[si][j] - y_ref) / np.linalg.norm(y_ref)
        print(f"stage {si} layer {li} {m}x{n}: x~ {e_xt:.2e}  y~ {e_yt:.2e}  y {e_y:.2e}", flush=True)
        li += 1

# ---- diagnosis of the first layer: per (row block, cell column) contributions
tiles, sm, sn, scale = info[0][0]
m, n = stages[0][0][0]
xt_p, yt_p = ctypes.c_void_p(), ctypes.c_void_p()
fn(chain._plan, 0, ctypes.byref(xt_p), ctypes.byref(yt_p))
npad, mpad = (n + 127) // 128 * 128, (m + 127) // 128 * 128
xt_t = torch.empty(npad * BP, dtype=torch.float16, device="cuda")
yt_t = torch.empty(B * mpad, dtype=torch.float32, device="cuda")
cp = lib.qtip_internal_copy
cp(ctypes.c_void_p(xt_t.data_ptr()), xt_p, npad * BP * 2)
cp(ctypes.c_void_p(yt_t.data_ptr()), yt_p, B * mpad * 4)
xt_g = xt_t.cpu().numpy().astype(np.float64).reshape(npad // 8, BP, 8).transpose(1, 0, 2).reshape(BP, npad)[:B, :n]
yt_g = yt_t.cpu().numpy().astype(np.float64).reshape(B, mpad)[:, :m]
W = gemv.dense_decode(tiles, p)
for rb in range(m // 128):
    g = yt_g[0, rb * 128:(rb + 1) * 128]
    line = []
    for rb2 in range(m // 128):
        for kc in range(n // 128):
            c = W[rb2 * 128:(rb2 + 1) * 128, kc * 128:(kc + 1) * 128] @ xt_g[0, kc * 128:(kc + 1) * 128]
            line.append(f"rb{rb2}kc{kc}:{np.dot(g, c) / (np.linalg.norm(g) * np.linalg.norm(c)):+.2f}")
    print(f"y~ rows of rb {rb}: cos with", " ".join(line), flush=True)
# the same layer through impl 7
lay = chain.layers[0]
qtip.set_matvec_impl(7)
y7 = lay(torch.from_numpy(x).cuda()).cpu().numpy()
qtip.set_matvec_impl(0)
print("impl 7 same layer vs chain y:", np.linalg.norm(y7 - outs[0][0]) / np.linalg.norm(y7))
