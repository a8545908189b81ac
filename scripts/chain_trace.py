#!/usr/bin/env python
"""Per-stage timeline of the chain kernel (globaltimer events of every CTA, see k_chain.cu CTR) on
the first `blocks` blocks of the 7B step.  Times in us from the kernel's first event.

usage: python scripts/chain_trace.py [code] [k] [blocks]
"""
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

code = sys.argv[1] if len(sys.argv) > 1 else "3inst"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
blocks = int(sys.argv[3]) if len(sys.argv) > 3 else 4
yld = int(sys.argv[4]) if len(sys.argv) > 4 else 1
lib = qtip.load()
lib.qtip_internal_set_chain_yield.argtypes = [ctypes.c_int]
lib.qtip_internal_set_chain_yield(yld)
VAR = {"3inst": 1.547, "1mad": 1.0, "hyb": 1.0}
lut = synth.gaussian_lut(9) if code == "hyb" else None
protos = {}
for si, (m, n) in enumerate([(4096, 4096), (11008, 4096), (4096, 11008)]):
    protos[(m, n)] = QTIPLinear(m, n, code=code, k=k).load_tiles(synth.random_tiles(m, n, k, seed=1000 + si),
                                                                  synth.random_sign_bytes(m, 3001 + si),
                                                                  synth.random_sign_bytes(n, 3000 + si),
                                                                  scale=1.0 / np.sqrt(n * VAR[code]), lut=lut)


def lay(m, n):
    pr = protos[(m, n)]
    l = QTIPLinear(m, n, code=code, k=k)
    l.packed.copy_(pr.packed)
    l.sign_m.copy_(pr.sign_m)
    l.sign_n.copy_(pr.sign_n)
    l.lut, l.scale = pr.lut, pr.scale
    return l


stages = []
for b in range(blocks):
    stages += [([lay(4096, 4096) for _ in range(3)], 0), ([lay(4096, 4096)], 0), ([lay(11008, 4096) for _ in range(2)], 0),
               ([lay(4096, 11008)], 0)]
chain = QTIPChain(stages, B=1)
x = torch.from_numpy(synth.random_x(1, 4096, seed=1)).cuda()
for _ in range(3):
    chain(x)
torch.cuda.synchronize()
P = torch.cuda.get_device_properties(0).multi_processor_count
KT = 160
tr = torch.zeros(2 * P * KT * 8, dtype=torch.int64, device="cuda")
fn = lib.qtip_internal_set_chain_trace
fn.argtypes = [ctypes.c_void_p]
assert fn(ctypes.c_void_p(tr.data_ptr())) == 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
chain(x)
e1.record()
torch.cuda.synchronize()
fn(ctypes.c_void_p(0))
ms = e0.elapsed_time(e1)
tt_all = tr.cpu().numpy().reshape(2, P, KT, 8).astype(np.float64)
t, tk = tt_all[0], tt_all[1]
ns_ = sum(len(s_[0]) for s_ in stages)
t0 = t[t > 0].min()
t = np.where(t > 0, (t - t0) / 1e3, np.nan)
print(f"yield={yld} {code} k={k}: {blocks} blocks, {ns_} stages, {sum(len(s[0]) for s in stages)} layers, kernel+memset {ms * 1e3:.1f} us "
      f"(traced), last event {np.nanmax(t):.1f} us")
names = ["q", "k", "v", "o", "gate", "up", "down"]
print("stage        win_wait(med)  win_land(med/max)  mma_done(med/max)  E_done(max)  T_start(min)  T_end(max)  dec_first(med)  prod_first(med)")
for s in range(min(ns_, KT)):
    col = lambda e: t[:, s, e]  # noqa: E731
    med = lambda v: np.nanmedian(v) if np.isfinite(v).any() else float("nan")  # noqa: E731
    mx = lambda v: np.nanmax(v) if np.isfinite(v).any() else float("nan")  # noqa: E731
    mn = lambda v: np.nanmin(v) if np.isfinite(v).any() else float("nan")  # noqa: E731
    print(f"{s:3d} {names[s % 7]:8s} {med(col(0)):9.1f}  {med(col(1)):9.1f}/{mx(col(1)):7.1f}  {med(col(2)):9.1f}/{mx(col(2)):7.1f}"
          f"  {mx(col(3)):9.1f}  {mn(col(4)):9.1f}  {mx(col(5)):9.1f}  {med(col(6)):9.1f}  {med(col(7)):9.1f}")

tk = np.where(tk > 0, (tk - t0) / 1e3, np.nan)
print("task phases (us after task start): CTA, transition, [D/sign fill, loads+acc, shuffles+reg, exchange+store, end, fence]")
shown = 0
for s_ in range(min(ns_ + 1, KT)):
    for c in range(P):
        v = tk[c, s_]
        if np.isfinite(v[0]) and shown < 40:
            print(c, s_, " ".join(f"{x - v[0]:7.2f}" for x in v[1:7]))
            shown += 1
