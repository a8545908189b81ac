#!/usr/bin/env python
"""Steady-state decode-GEMV rate (weights / clock / SM) of a matvec impl on one tall layer, where
per-launch ramp and tail are negligible: graph of R replays of one m x n layer (RHT-in only, the
GEMV output is scale * W~ x~), minus the same graph for a small layer of the same n.

usage: python scripts/gemv_rate.py impl [code] [k] [m] [n] [B]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2406_11235_b200 import qtip  # noqa: E402
from paper_2406_11235_b200.layer import QTIPLinear  # noqa: E402

impl = int(sys.argv[1]) if len(sys.argv) > 1 else 0
code = sys.argv[2] if len(sys.argv) > 2 else "3inst"
k = int(sys.argv[3]) if len(sys.argv) > 3 else 2
m = int(sys.argv[4]) if len(sys.argv) > 4 else 37888
n = int(sys.argv[5]) if len(sys.argv) > 5 else 4096
B = int(sys.argv[6]) if len(sys.argv) > 6 else 1
qtip.load(os.environ.get("QTIP_LIB", qtip.LIB_PATH))
qtip.set_matvec_impl(impl)
lut = synth.gaussian_lut(9) if code == "hyb" else None
sms = torch.cuda.get_device_properties(0).multi_processor_count


def layer_time(mm):
    lay = QTIPLinear(mm, n, code=code, k=k).load_tiles(synth.random_tiles(mm, n, k, seed=5),
                                                        synth.random_sign_bytes(mm, 1), synth.random_sign_bytes(n, 2),
                                                        lut=lut)
    x = torch.from_numpy(synth.random_x(B, n, seed=3)).cuda()
    y = torch.empty((B, mm), device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        lay.forward(x, out=y, flags=qtip.QTIP_RHT_IN)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(5):
                lay.forward(x, out=y, flags=qtip.QTIP_RHT_IN)
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
    return e0.elapsed_time(e1) / 50 * 1e3       # us per call


t_big = layer_time(m)
m_small = int(sys.argv[7]) if len(sys.argv) > 7 else m // 2
t_small = layer_time(m_small)
clk = 1.965e3                                   # MHz (bench clocks line: 1965 MHz under load)
dw = (m - m_small) * n
rate = dw / ((t_big - t_small) * clk) / sms
print(f"impl={impl} {code} k={k} n={n} B={B}: {m}x{n} {t_big:.1f} us, {m_small}x{n} {t_small:.1f} us -> "
      f"{rate:.1f} weights/clk/SM steady state ({dw * k / 8 / ((t_big - t_small) * 1e-6) / 1e9:.0f} GB/s)")
