#!/usr/bin/env python
"""GPU quantizer throughput (qtip_viterbi_tailbite, Algorithm 4) vs the CPU oracle's binary32 DP
(single thread) on the same seeded sequences.  usage: python scripts/viterbi_bench.py [code] [k] [nseq] [T]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from oracle import codes, viterbi  # noqa: E402
from paper_2406_11235_b200.quantize import QTIPQuantizer  # noqa: E402

code = sys.argv[1] if len(sys.argv) > 1 else "3inst"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
nseq = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
T = int(sys.argv[4]) if len(sys.argv) > 4 else 256
V = 2 if code == "hyb" else 1
lut = synth.gaussian_lut(9, 4000) if code == "hyb" else None
tab = codes.code_table(code, 16, lut=lut, Q=9) if code == "hyb" else codes.code_table(code, 16)
src = (synth.gaussian_source(nseq, T, seed=5000).astype(np.float32) * np.float32(tab.std())).astype(np.float32)
q = QTIPQuantizer(code, k, lut=lut)
d = torch.from_numpy(src).cuda()
q.encode(d[:8].contiguous())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
st, cost = q.encode(d)
e1.record()
torch.cuda.synchronize()
gpu_s = e0.elapsed_time(e1) / 1e3
ncpu = 4 if k * V <= 4 else 1
os.environ.setdefault("OMP_NUM_THREADS", "1")
t0 = time.perf_counter()
viterbi.tailbite_encode_f32_batch(src[:ncpu], 16, k, V, tab.astype(np.float32))
cpu_s = (time.perf_counter() - t0) / ncpu
print(f"{code} k={k} T={T}: GPU {nseq} sequences in {gpu_s * 1e3:.1f} ms = {gpu_s / nseq * 1e6:.1f} us/sequence "
      f"({nseq / gpu_s:.0f} seq/s, {nseq * T / gpu_s / 1e6:.2f} M weights/s); CPU oracle (binary32 DP, OMP threads="
      f"{os.environ.get('OMP_NUM_THREADS')}) {cpu_s * 1e3:.0f} ms/sequence; mean MSE/weight "
      f"{float(cost.mean()) / T / tab.std() ** 2:.4f}")
