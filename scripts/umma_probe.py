#!/usr/bin/env python
"""Quick check of the stream-K tcgen05 GEMV (impl 7): small layers of every code against the oracle,
then per-layer times (graph of 20 calls, RHT in/out) of impl 7 vs the round-1 kernels on the 7B shapes.

usage: python scripts/umma_probe.py [check|time|both]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2406_11235_b200 import qtip  # noqa: E402
from paper_2406_11235_b200.layer import QTIPLinear  # noqa: E402

qtip.load()
what = sys.argv[1] if len(sys.argv) > 1 else "both"


def check():
    from oracle import gemv
    for code, k in [("3inst", 2), ("1mad", 2), ("hyb", 4), ("hyb", 3), ("3inst", 3), ("1mad", 4), ("hyb", 2)]:
        for (m, n, B) in [(256, 256, 1), (384, 768, 1), (272, 336, 2), (1024, 512, 4), (256, 512, 16), (256, 256, 64)]:
            lut = synth.gaussian_lut(9) if code == "hyb" else None
            tiles = synth.random_tiles(m, n, k, seed=11 + k)
            sm, sn = synth.random_sign_bytes(m, 3001), synth.random_sign_bytes(n, 3000)
            lay = QTIPLinear(m, n, code=code, k=k).load_tiles(tiles, sm, sn, scale=0.37, lut=lut)
            x = synth.random_x(B, n, seed=2000 + B)
            qtip.set_matvec_impl(7)
            y = lay(torch.from_numpy(x).cuda()).cpu().numpy()
            qtip.set_matvec_impl(0)
            W = gemv.dense_decode(tiles, gemv.Params(k=k, V=2 if code == "hyb" else 1, code=code, lut=lut))
            ref = gemv.matvec(W, x.astype(np.float64), sn, sm, scale=0.37)
            err = float(np.linalg.norm(y - ref) / np.linalg.norm(ref))
            print(f"check {code} k={k} {m}x{n} B={B}: rel L2 {err:.2e} {'OK' if err < 1e-3 else 'FAIL'}", flush=True)


def layer_us(impl, code, k, m, n, B=1, flags=3, reps=20):
    lut = synth.gaussian_lut(9) if code == "hyb" else None
    lays = [QTIPLinear(m, n, code=code, k=k).load_tiles(synth.random_tiles(m, n, k, seed=5 + i),
                                                         synth.random_sign_bytes(m, 1), synth.random_sign_bytes(n, 2),
                                                         lut=lut) for i in range(4)]
    x = torch.from_numpy(synth.random_x(B, n, seed=3)).cuda()
    y = torch.empty((B, m), device="cuda")
    qtip.set_matvec_impl(impl)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    try:
        with torch.cuda.stream(s):
            for l in lays:
                l.forward(x, out=y, flags=flags)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for i in range(reps):
                    lays[i % 4].forward(x, out=y, flags=flags)
    finally:
        qtip.set_matvec_impl(0)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (10 * reps) * 1e3


def timing():
    for code, k in [("3inst", 2), ("hyb", 4)]:
        for (m, n) in [(4096, 4096), (11008, 4096), (4096, 11008), (37888, 4096)]:
            row = []
            for impl in (7, 3, 4, 6):
                try:
                    us = layer_us(impl, code, k, m, n)
                    us1 = layer_us(impl, code, k, m, n, flags=1)
                    row.append(f"impl{impl} {us:7.2f} us ({m * n * k / 8 / us / 1e3:6.0f} GB/s) gemv+red {us1:7.2f}")
                except Exception as e:                                 # noqa: BLE001
                    row.append(f"impl{impl} err {str(e)[:60]}")
            print(f"{code} k={k} {m}x{n}: " + " | ".join(row), flush=True)


if what in ("check", "both"):
    check()
if what in ("time", "both"):
    timing()
