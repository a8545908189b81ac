#!/usr/bin/env python
"""Small workload touching every libqtip kernel, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): decode, RHT forward / inverse, every matvec implementation (1-7) for each
code at batch 1 and 3 (and 16 where supported), the grouped launches (impl 6 and 7) and the GPU
quantizer.  Exits non-zero if a result differs from the oracle.

usage: compute-sanitizer --tool memcheck python scripts/sanitize_run.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from oracle import gemv  # noqa: E402
from paper_2406_11235_b200 import qtip  # noqa: E402
from paper_2406_11235_b200.layer import QTIPLinear, forward_group  # noqa: E402

qtip.load()
torch.cuda.set_device(0)
bad = 0


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


m, n = 384, 768
for code, k in [("3inst", 2), ("1mad", 2), ("hyb", 4), ("hyb", 3)]:
    lut = synth.gaussian_lut(9) if code == "hyb" else None
    tiles = synth.random_tiles(m, n, k, seed=9)
    sm, sn = synth.random_sign_bytes(m, 1), synth.random_sign_bytes(n, 2)
    lay = QTIPLinear(m, n, code=code, k=k).load_tiles(tiles, sm, sn, scale=0.5, lut=lut)
    W = gemv.dense_decode(tiles, gemv.Params(k=k, V=2 if code == "hyb" else 1, code=code, lut=lut))
    dec = lay.decode().cpu().numpy().view(np.uint16)
    bad += int(not np.array_equal(dec, W.astype(np.float16).view(np.uint16)))
    for impl in range(1, 8):
        for B in (1, 3, 16):
            if impl in (4, 5, 6) and B > 4:
                continue
            if impl != 1 and impl != 7 and k == 1:
                continue
            x = synth.random_x(B, n, seed=3 + B)
            qtip.set_matvec_impl(impl)
            try:
                y = lay(torch.from_numpy(x).cuda()).cpu().numpy()
            except qtip.QtipError as e:
                print(f"impl {impl} {code} k={k} B={B}: {e}")
                continue
            finally:
                qtip.set_matvec_impl(0)
            err = rel(y, gemv.matvec(W, x.astype(np.float64), sn, sm, scale=0.5))
            print(f"impl {impl} {code} k={k} B={B}: rel L2 {err:.2e}", flush=True)
            bad += int(err > 1e-3)
    # grouped launches (persistent impl 6 grouping; the stream-K kernel with the group's cells)
    layers = [QTIPLinear(m, n, code=code, k=k).load_tiles(synth.random_tiles(m, n, k, seed=20 + g), sm, sn, lut=lut)
              for g in range(3)]
    x = torch.from_numpy(synth.random_x(1, n, seed=5)).cuda()
    for impl in (6, 7):
        qtip.set_matvec_impl(impl)
        try:
            ys = [o.cpu().numpy() for o in forward_group(layers, x)]
        finally:
            qtip.set_matvec_impl(0)
        for g in range(3):
            Wg = gemv.dense_decode(synth.random_tiles(m, n, k, seed=20 + g),
                                   gemv.Params(k=k, V=2 if code == "hyb" else 1, code=code, lut=lut))
            err = rel(ys[g], gemv.matvec(Wg, x.cpu().numpy().astype(np.float64), sn, sm))
            bad += int(err > 1e-3)
        print(f"grouped impl {impl} {code} k={k}: ok", flush=True)

# the GPU quantizer (Algorithm 4)
from oracle import codes, viterbi  # noqa: E402
from paper_2406_11235_b200.quantize import QTIPQuantizer  # noqa: E402
tab = codes.code_table("3inst", 16)
src = (synth.gaussian_source(4, 32, seed=5000).astype(np.float32) * np.float32(tab.std())).astype(np.float32)
st, cost = QTIPQuantizer("3inst", 2).encode(torch.from_numpy(src).cuda())
ref_st, _ = viterbi.tailbite_encode_f32_batch(src, 16, 2, 1, tab.astype(np.float32))
bad += int(not np.array_equal(st.cpu().numpy().view(np.uint32), ref_st))
torch.cuda.synchronize()
print("sanitize_run:", "FAILED" if bad else "ok", bad)
sys.exit(1 if bad else 0)
