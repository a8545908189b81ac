#!/usr/bin/env python
"""Per-layer time breakdown in CUDA graphs (warm L2 for x / signs, weights streamed from HBM).

For each Llama-2-7B shape: full layer (RHT-in, GEMV, reduce, RHT-out), matvec without RHT
(convert, GEMV, reduce), RHT alone for n and for m.  Each graph holds R distinct layers of the
shape (R * bytes > L2) and is replayed; time / (replays * R).
usage: python scripts/layer_breakdown.py [code] [k] [B] [pdl 0/1]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2406_11235_b200 import qtip  # noqa: E402
from paper_2406_11235_b200.layer import QTIPLinear  # noqa: E402

code = sys.argv[1] if len(sys.argv) > 1 else "3inst"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
pdl = int(sys.argv[4]) if len(sys.argv) > 4 else 1
impl = int(sys.argv[5]) if len(sys.argv) > 5 else 0
qtip.load()
qtip.set_matvec_impl(impl)
qtip.set_pdl(bool(pdl))
dev = torch.device("cuda", 0)
lut = synth.gaussian_lut(9) if code == "hyb" else None


def timed(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / reps


for (m, n) in [(4096, 4096), (11008, 4096), (4096, 11008)]:
    R = max(2, int(300e6 // (m * n * k // 8)))
    tiles = synth.random_tiles(m, n, k, seed=7)
    sm, sn = synth.random_sign_bytes(m, 1), synth.random_sign_bytes(n, 2)
    proto = QTIPLinear(m, n, code=code, k=k, device=dev).load_tiles(tiles, sm, sn, lut=lut)
    layers = []
    for _ in range(R):
        l = QTIPLinear(m, n, code=code, k=k, device=dev)
        l.packed.copy_(proto.packed); l.sign_m.copy_(proto.sign_m); l.sign_n.copy_(proto.sign_n)
        l.lut = proto.lut
        layers.append(l)
    x = torch.from_numpy(synth.random_x(B, n, seed=3)).to(dev)
    y = torch.empty((B, m), device=dev)
    full = timed(lambda: [l.forward(x, out=y) for l in layers]) / R
    bare = timed(lambda: [l.forward(x, out=y, flags=0) for l in layers]) / R
    xo = torch.empty_like(x)
    yo = torch.empty_like(y)
    rin = timed(lambda: [qtip.qtip_rht(n, B, layers[0].sign_n, x, xo) for _ in range(R)]) / R
    rout = timed(lambda: [qtip.qtip_rht(m, B, layers[0].sign_m, y, yo, inverse=True) for _ in range(R)]) / R
    gb = m * n * k / 8
    print(f"impl={impl} {code} k={k} B={B} pdl={pdl} {m}x{n}: layer {full:7.2f} us ({gb / full / 1e3:6.1f} GB/s) | "
          f"no-RHT matvec {bare:7.2f} us ({gb / bare / 1e3:6.1f} GB/s) | rht(n) {rin:6.2f} | rht_inv(m) {rout:6.2f}",
          flush=True)
    del layers, proto
    torch.cuda.empty_cache()
