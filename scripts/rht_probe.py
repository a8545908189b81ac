#!/usr/bin/env python
"""Run qtip_rht forward + inverse for a few orders (for ncu captures of the RHT kernel)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2406_11235_b200 import qtip  # noqa: E402

qtip.load()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for n in [4096, 11008, 28672]:
    s = torch.from_numpy(synth.random_sign_bytes(n, 1)).cuda()
    x = torch.from_numpy(synth.random_x(B, n, seed=2)).cuda()
    y, z = torch.empty_like(x), torch.empty_like(x)
    for _ in range(3):
        qtip.qtip_rht(n, B, s, x, y)
        qtip.qtip_rht(n, B, s, y, z, inverse=True)
    torch.cuda.synchronize()
    print(n, float((z - x).abs().max()))
