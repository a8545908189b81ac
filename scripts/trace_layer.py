#!/usr/bin/env python
"""CTA timeline of consecutive layer forwards (RHT-in -> GEMV -> RHT-out) in one CUDA graph.

usage: python scripts/trace_layer.py m n [code] [k] [layers] [pdl]
Prints, per kernel launch: kind, CTAs, first entry, PDL-wait release (min/median/max), exit
(min/median/max), all in us relative to the first recorded entry.
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
NL = int(sys.argv[5]) if len(sys.argv) > 5 else 3
pdl = int(sys.argv[6]) if len(sys.argv) > 6 else 1
fused = int(sys.argv[7]) if len(sys.argv) > 7 else 0
impl = int(sys.argv[8]) if len(sys.argv) > 8 else 0
lib = qtip.load()
lib.qtip_internal_set_knob(1, fused)
qtip.set_matvec_impl(impl)
qtip.set_pdl(bool(pdl))
lib.qtip_internal_set_cta_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
lut = synth.gaussian_lut(9) if code == "hyb" else None
layers = [QTIPLinear(m, n, code=code, k=k).load_tiles(synth.random_tiles(m, n, k, seed=7 + i),
                                                      synth.random_sign_bytes(m, 1), synth.random_sign_bytes(n, 2),
                                                      lut=lut) for i in range(NL)]
x = torch.from_numpy(synth.random_x(1, n, seed=3)).cuda()
y = torch.empty((1, m), device="cuda")
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
CAP = 200000
buf = torch.zeros(1 + 8 * CAP, dtype=torch.int64, device="cuda")
assert lib.qtip_internal_set_cta_trace(buf.data_ptr(), CAP) == 0
g.replay()
torch.cuda.synchronize()
assert lib.qtip_internal_set_cta_trace(None, 0) == 0
b = buf.cpu().numpy()
cnt = min(int(b[0]), CAP)
r = b[1:1 + 8 * cnt].reshape(cnt, 8).astype(np.int64)
t_ref = r[:, 3].min()
names = {1: "rht_in", 2: "rht_out", 3: "gemv", 4: "gemv_row"}
units = r[:, 0] >> 8                        # gemv: cells processed by the CTA
r[:, 0] &= 0xFF
# split each kind's records into launches at gaps between sorted entry times
out = []
for tag in sorted(set(r[:, 0])):
    q = np.concatenate([r, units[:, None]], axis=1)[r[:, 0] == tag]
    q = q[np.argsort(q[:, 3])]
    cuts = np.where(np.diff(q[:, 3]) > 2000)[0] + 1
    for part in np.split(q, cuts):
        out.append((part[:, 3].min(), tag, part))
print(f"{m}x{n} {code} k={k} layers={NL} pdl={pdl}: {cnt} CTA records")
for t0, tag, p in sorted(out, key=lambda z: z[0]):
    e, w, x_ = (p[:, 3] - t_ref) / 1e3, (p[:, 4] - t_ref) / 1e3, (p[:, 5] - t_ref) / 1e3
    print(f"  {names.get(int(tag), tag):8s} ctas={len(p):5d} entry {e.min():7.2f}..{e.max():7.2f}  "
          f"wait-release {w.min():7.2f}/{np.median(w):7.2f}/{w.max():7.2f}  "
          f"exit {x_.min():7.2f}/{np.median(x_):7.2f}/{x_.max():7.2f}  sms={len(set(p[:, 2]))}"
          + (f"  cells/cta {p[:, 8].min()}..{p[:, 8].max()} (sum {p[:, 8].sum()})" if tag in (3, 4) else ""))
    if tag in (3, 4):
        late = p[np.argsort(p[:, 5])[-5:]]
        for z in late:
            red = f" last reduce RB {z[7]-1} at {(z[6]-t_ref)/1e3:7.2f}" if z[7] else ""
            print(f"      late cta {z[1]:5d} sm {z[2]:3d} cells {z[8]} entry {(z[3]-t_ref)/1e3:7.2f} exit {(z[5]-t_ref)/1e3:7.2f}{red}")
        rr = p[p[:, 7] > 0]
        if len(rr):
            ts = (rr[:, 6] - t_ref) / 1e3
            print(f"      reductions: {len(rr)} CTAs, last-reduce start {ts.min():7.2f}/{np.median(ts):7.2f}/{ts.max():7.2f}, "
                  f"reducer exit median {np.median((rr[:, 5]-t_ref)/1e3):7.2f}")
