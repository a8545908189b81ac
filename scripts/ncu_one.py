#!/usr/bin/env python
"""One layer called a few times, for ncu: python scripts/ncu_one.py impl code k m n [B] [flags]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2406_11235_b200 import qtip  # noqa: E402
from paper_2406_11235_b200.layer import QTIPLinear  # noqa: E402

impl, code, k, m, n = int(sys.argv[1]), sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
B = int(sys.argv[6]) if len(sys.argv) > 6 else 1
flags = int(sys.argv[7]) if len(sys.argv) > 7 else 3
qtip.load()
qtip.set_matvec_impl(impl)
lut = synth.gaussian_lut(9) if code == "hyb" else None
lay = QTIPLinear(m, n, code=code, k=k).load_tiles(synth.random_tiles(m, n, k, seed=5), synth.random_sign_bytes(m, 1),
                                                   synth.random_sign_bytes(n, 2), lut=lut)
x = torch.from_numpy(synth.random_x(B, n, seed=3)).cuda()
for _ in range(4):
    y = lay(x, flags=flags)
torch.cuda.synchronize()
print("done", float(y.abs().sum()))
