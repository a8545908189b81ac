#!/usr/bin/env python
"""Time qtip_rht (forward and inverse, fp32 out) per call for the 7B / 70B orders and batch widths:
a CUDA graph of 50 back-to-back calls, CUDA events.

usage: python scripts/rht_bench.py [B list, comma-separated] [n list, comma-separated]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2406_11235_b200 import qtip  # noqa: E402

qtip.load()
Bs = [int(b) for b in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 2, 4, 8, 16]
R = 50
st = torch.cuda.Stream()
Ns = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [4096, 11008, 8192, 28672]
for n in Ns:
    for B in Bs:
        s = torch.from_numpy(synth.random_sign_bytes(n, 1)).cuda()
        x = torch.from_numpy(synth.random_x(B, n, seed=2)).cuda()
        y = torch.empty_like(x)
        res = []
        for inv in (0, 1):
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                qtip.qtip_rht(n, B, s, x, y, inverse=bool(inv))
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    for _ in range(R):
                        qtip.qtip_rht(n, B, s, x, y, inverse=bool(inv))
            torch.cuda.current_stream().wait_stream(st)
            g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            res.append(1e3 * e0.elapsed_time(e1) / (5 * R))
        print(f"n={n:6d} B={B:3d}: forward {res[0]:7.2f} us  inverse {res[1]:7.2f} us", flush=True)
