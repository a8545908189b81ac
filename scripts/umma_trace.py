#!/usr/bin/env python
"""CTA 0 timeline of the stream-K tcgen05 GEMV (k_umma.cu debug trace, clock64 cycles).

usage: python scripts/umma_trace.py code k m n [B]
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

code, k, m, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
B = int(sys.argv[5]) if len(sys.argv) > 5 else 1
lib = qtip.load()
qtip.set_matvec_impl(int(os.environ.get("IMPL", "7")))
lut = synth.gaussian_lut(9) if code == "hyb" else None
lay = QTIPLinear(m, n, code=code, k=k).load_tiles(synth.random_tiles(m, n, k, seed=5), synth.random_sign_bytes(m, 1),
                                                   synth.random_sign_bytes(n, 2), lut=lut)
x = torch.from_numpy(synth.random_x(B, n, seed=3)).cuda()
buf = torch.zeros(16 * 64, dtype=torch.int64, device="cuda")
for _ in range(3):
    lay(x)
torch.cuda.synchronize()
lib.qtip_internal_set_umma_trace.argtypes = [ctypes.c_void_p]
lib.qtip_internal_set_umma_trace_cta(int(os.environ.get("TRACE_CTA", "0")))
lib.qtip_internal_set_umma_trace(ctypes.c_void_p(buf.data_ptr()))
lay(x)
torch.cuda.synchronize()
lib.qtip_internal_set_umma_trace(None)
t = buf.cpu().numpy().reshape(16, 64).astype(np.int64)
t0 = t[7, 0]
names = ["prod issue", "dec full", "dec aempty", "dec handoff", "mma afull", "mma issued", "epi dfull"]
print(f"misc: start 0, x~ ready {t[7,1]-t0}, end {t[7,2]-t0}")
print("cell grp  full-seen  aempty-ok  handoff | x-issued  x-seen  mma-seen  mma-issued | decode  mma-issue")
for c in range(64):
    if not t[3, c]:
        continue
    r = [int(t[kk, c] - t0) if t[kk, c] else -1 for kk in (1, 2, 3, 9, 8, 4, 5)]
    print(f"{c:4d} {c % 3:3d} {r[0]:10d} {r[1]:10d} {r[2]:8d} | {r[3]:8d} {r[4]:7d} {r[5]:9d} {r[6]:11d} | "
          f"{r[2]-r[1]:6d} {r[6]-r[5]:6d}")
print("epilogue segments:", " ".join(str(int(v - t0)) for v in t[6] if v))
