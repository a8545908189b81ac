#!/usr/bin/env python
"""Per-stage times of the 7B block (graph of 32 replicas of one stage, CUDA events): grouped q,k,v,
o, grouped gate,up, down -- full (RHT-in, GEMV, RHT-out) and GEMV only (x~ ready, RHT-out off).

usage: python scripts/stage_breakdown.py [code] [k] [B] [matvec impl for the single layers]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2406_11235_b200 import qtip  # noqa: E402
from paper_2406_11235_b200.layer import QTIPLinear, forward_group  # noqa: E402

code = sys.argv[1] if len(sys.argv) > 1 else "3inst"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
impl = int(sys.argv[4]) if len(sys.argv) > 4 else 0
qtip.load()
qtip.set_matvec_impl(impl)
lut = synth.gaussian_lut(9) if code == "hyb" else None
R = 32


def make(m, n, i):
    return QTIPLinear(m, n, code=code, k=k).load_tiles(synth.random_tiles(m, n, k, seed=i), synth.random_sign_bytes(m, i),
                                                       synth.random_sign_bytes(n, i + 1), lut=lut)


stages = {"qkv (grouped)": [(4096, 4096)] * 3, "o": [(4096, 4096)], "gate,up (grouped)": [(11008, 4096)] * 2,
          "down": [(4096, 11008)]}
s = torch.cuda.Stream()
for name, shp in stages.items():
    reps = [[make(m, n, 10 * r + j) for j, (m, n) in enumerate(shp)] for r in range(R)]
    n = shp[0][1]
    x = torch.from_numpy(synth.random_x(B, n, seed=1)).cuda()
    outs = [[torch.empty((B, m), device="cuda") for (m, _) in shp] for _ in range(R)]
    res = {}
    for label, flags in (("full", qtip.QTIP_RHT_IN | qtip.QTIP_RHT_OUT), ("gemv", qtip.QTIP_RHT_IN | qtip.QTIP_XT_READY)):
        def run():
            for ls, os_ in zip(reps, outs):
                if len(ls) > 1:
                    forward_group(ls, x, outs=os_, flags=flags)
                else:
                    ls[0].forward(x, out=os_[0], flags=flags)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            if label == "gemv":
                for ls, os_ in zip(reps, outs):           # x~ into every workspace first
                    if len(ls) > 1:
                        forward_group(ls, x, outs=os_)
                    else:
                        ls[0].forward(x, out=os_[0])
            run()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                run()
        torch.cuda.current_stream().wait_stream(s)
        for _ in range(3):
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        res[label] = 1e3 * e0.elapsed_time(e1) / (10 * R)
    nbytes = sum(m * n * k // 8 for (m, n) in shp)
    print(f"{code} k={k} B={B} impl={impl} {name:18s}: full {res['full']:7.2f} us  gemv-only {res['gemv']:7.2f} us  "
          f"({nbytes / res['gemv'] / 1e3:7.1f} GB/s gemv)  rht+boundaries {res['full'] - res['gemv']:6.2f} us")
    del reps
    torch.cuda.empty_cache()
