#!/usr/bin/env python
"""Per-stage times of the 7B block with each transform switched on/off (graph of 32 replicas of one
stage, CUDA events): full (RHT-in, GEMV, RHT-out), in+gemv, gemv+out, gemv only -- locates the cost of
the kernel boundaries around the decode-GEMV.

usage: python scripts/stage_flags.py [code] [k] [B] [matvec impl] [stages, comma-separated]
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
only = sys.argv[5].split(",") if len(sys.argv) > 5 else None
qtip.load()
qtip.set_matvec_impl(impl)
if os.environ.get("QTIP_L2_PREFETCH") is not None:
    qtip.load().qtip_internal_set_knob(4, int(os.environ["QTIP_L2_PREFETCH"]))
lut = synth.gaussian_lut(9) if code == "hyb" else None
R = 32


def make(m, n, i):
    return QTIPLinear(m, n, code=code, k=k).load_tiles(synth.random_tiles(m, n, k, seed=i), synth.random_sign_bytes(m, i),
                                                       synth.random_sign_bytes(n, i + 1), lut=lut)


IN, OUT, XR = qtip.QTIP_RHT_IN, qtip.QTIP_RHT_OUT, qtip.QTIP_XT_READY
modes = (("full", IN | OUT), ("in+gemv", IN), ("gemv+out", IN | XR | OUT), ("gemv", IN | XR))
stages = {"qkv": [(4096, 4096)] * 3, "o": [(4096, 4096)], "gateup": [(11008, 4096)] * 2, "down": [(4096, 11008)],
          "big": [(12288, 4096)]}
s = torch.cuda.Stream()
for name, shp in stages.items():
    if (only and name not in only) or (not only and name == "big"):
        continue
    reps = [[make(m, n, 10 * r + j) for j, (m, n) in enumerate(shp)] for r in range(R)]
    if code == "hyb":                                   # one LUT per group, as bench.py (the grouped launch)
        for ls in reps:
            for l_ in ls[1:]:
                l_.lut = ls[0].lut
    n = shp[0][1]
    x = torch.from_numpy(synth.random_x(B, n, seed=1)).cuda()
    outs = [[torch.empty((B, m), device="cuda") for (m, _) in shp] for _ in range(R)]
    res = {}
    for label, flags in modes:
        def run(fl):
            for ls, os_ in zip(reps, outs):
                if len(ls) > 1:
                    forward_group(ls, x, outs=os_, flags=fl)
                else:
                    ls[0].forward(x, out=os_[0], flags=fl)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            run(IN | OUT)                                   # x~ into every workspace first
            run(flags)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                run(flags)
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
    print(f"{code} k={k} B={B} impl={impl} {name:7s}: " + "  ".join(f"{lb} {v:7.2f}" for lb, v in res.items()) +
          f"  us  (gemv {nbytes / res['gemv'] / 1e3:7.1f} GB/s)", flush=True)
    del reps
    torch.cuda.empty_cache()
