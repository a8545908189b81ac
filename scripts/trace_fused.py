#!/usr/bin/env python
"""Phase timeline of the fused single-launch layer kernel (impl 5) for consecutive layers in one
CUDA graph: per launch, the min / median / max over CTAs of each phase mark (k_layer.cu
trace_mark), in us relative to the first CTA entry of the first traced launch.

usage: python scripts/trace_fused.py m n [code] [k] [layers] [B]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2406_11235_b200 import qtip  # noqa: E402
from paper_2406_11235_b200.layer import QTIPLinear  # noqa: E402

m, n = int(sys.argv[1]), int(sys.argv[2])
code = sys.argv[3] if len(sys.argv) > 3 else "3inst"
k = int(sys.argv[4]) if len(sys.argv) > 4 else 2
NL = int(sys.argv[5]) if len(sys.argv) > 5 else 4
B = int(sys.argv[6]) if len(sys.argv) > 6 else 1
debug = int(sys.argv[7]) if len(sys.argv) > 7 else 0
pdl = int(sys.argv[8]) if len(sys.argv) > 8 else 1
impl = int(sys.argv[9]) if len(sys.argv) > 9 else 5
lib = qtip.load()
lib.qtip_internal_set_knob(2, debug)
qtip.set_pdl(bool(pdl))
qtip.set_matvec_impl(impl)
lib.qtip_internal_set_layer_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
lut = synth.gaussian_lut(9) if code == "hyb" else None
layers = [QTIPLinear(m, n, code=code, k=k).load_tiles(synth.random_tiles(m, n, k, seed=7 + i),
                                                      synth.random_sign_bytes(m, 1), synth.random_sign_bytes(n, 2),
                                                      lut=lut) for i in range(NL)]
x = torch.from_numpy(synth.random_x(B, n, seed=3)).cuda()
y = torch.empty((B, m), device="cuda")
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for l in layers:
        l.forward(x, out=y)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for l in layers:
            l.forward(x, out=y)
torch.cuda.current_stream().wait_stream(s)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
cap = 148 * NL * 2
buf = torch.zeros(1 + 14 * cap, dtype=torch.int64, device="cuda")
lib.qtip_internal_set_layer_trace(ctypes.c_void_p(buf.data_ptr()), cap)
g.replay()
torch.cuda.synchronize()
lib.qtip_internal_set_layer_trace(None, 0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    g.replay()
e1.record()
torch.cuda.synchronize()
print(f"{m}x{n} {code} k={k} B={B}: {1e3 * e0.elapsed_time(e1) / (10 * NL):.2f} us/layer (untraced graph)")
b = buf.cpu().numpy()
cnt = int(b[0])
rec = b[1:1 + 14 * cnt].reshape(cnt, 14)
t = rec[:, 2:].astype(np.float64)
# launches: CTAs sorted by entry time, split into groups of grid size
order = np.argsort(t[:, 0])
t = t[order]
P = 148
t0 = t[:, 0].min()
names = ["entry", "pdl", "staged", "fwht", "x~", "gemv", "red", "prol/sh", "bar2", "ystg", "fwho", "exit"]
if debug & 4:                                   # SM clock64 marks: per-CTA cycles since its PDL release
    raw = rec[:, 2:].astype(np.float64)
    print(f"  part_smem {int(rec[0, 1]) >> 32 & 0xff}  ring stages {int(rec[0, 1]) >> 40}")
    for j, nm in enumerate(names):
        ok = (raw[:, j] > 0) & (raw[:, 1] > 0)
        if ok.any():
            d = raw[ok, j] - raw[ok, 1]
            print(f"  {nm:8s} cycles after pdl release: median {np.median(d):8.0f}  max {np.max(d):8.0f}")
    sys.exit(0)
for li in range(NL):
    tl = (t[li * P:(li + 1) * P] - t0) / 1e3
    cols = []
    for j, nm in enumerate(names):
        v = tl[:, j]
        v = v[v > -1e6]
        if len(v):
            cols.append(f"{nm} {np.median(v):6.2f}/{np.max(v):6.2f}")
    print(f"launch {li}: " + " | ".join(cols))
