#!/usr/bin/env python
"""Run a few full layer forwards of one shape (for ncu captures).  usage: gemv_probe.py m n [code] [k] [B]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2406_11235_b200 import qtip  # noqa: E402
from paper_2406_11235_b200.layer import QTIPLinear  # noqa: E402

m, n = int(sys.argv[1]), int(sys.argv[2])
code = sys.argv[3] if len(sys.argv) > 3 else "3inst"
k = int(sys.argv[4]) if len(sys.argv) > 4 else 2
B = int(sys.argv[5]) if len(sys.argv) > 5 else 1
qtip.load()
lut = synth.gaussian_lut(9) if code == "hyb" else None
lay = QTIPLinear(m, n, code=code, k=k).load_tiles(synth.random_tiles(m, n, k, seed=7), synth.random_sign_bytes(m, 1),
                                                  synth.random_sign_bytes(n, 2), lut=lut)
x = torch.from_numpy(synth.random_x(B, n, seed=3)).cuda()
for _ in range(5):
    y = lay(x)
torch.cuda.synchronize()
print(y.shape, float(y.abs().sum()))
