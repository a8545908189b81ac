#!/usr/bin/env python
"""Cycles of one chain transform task run alone (1 CTA of 128 threads): 4096 inverse / forward /
fused, 11008 inverse / forward.  usage: python scripts/xform_bench.py"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2406_11235_b200 import qtip  # noqa: E402
from paper_2406_11235_b200.layer import QTIPChain, QTIPLinear  # noqa: E402

lib = qtip.load()
fn = lib.qtip_internal_chain_xform_bench
fn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
               ctypes.c_void_p]


def L(m, n):
    return QTIPLinear(m, n, code="3inst", k=2).load_tiles(synth.random_tiles(m, n, 2, seed=1), synth.random_sign_bytes(m, 2),
                                                           synth.random_sign_bytes(n, 3), scale=0.01)


stages = [([L(4096, 4096)], 0), ([L(11008, 4096)], 0), ([L(4096, 11008)], 0), ([L(4096, 4096)], 0)]
ch = QTIPChain(stages, B=1)
x = torch.from_numpy(synth.random_x(1, 4096, seed=1)).cuda()
ch(x)
torch.cuda.synchronize()
out = torch.zeros(1, dtype=torch.int64, device="cuda")
for name, li, d, part, fu in [("4096 fwd (x)", 0, 0, 0, 0), ("4096 inv", 0, 1, 0, 0), ("11008 inv part 0", 1, 1, 0, 0),
                              ("11008 fwd part 0", 2, 0, 0, 0), ("4096 fwd fused", 3, 0, 0, 1), ("4096 fwd from y", 3, 0, 0, 0)]:
    for iters in (1, 10):
        rc = fn(ch._plan, li, d, part, fu, iters, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(x.data_ptr()))
        assert rc == 0, rc
        print(f"{name:20s} iters {iters:2d}: {out.item() / iters:9.0f} cycles/task", flush=True)
