#!/usr/bin/env python
"""Compare CUDA-event GEMV timing (graph event nodes, PDL off) with the CTA timeline."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2406_11235_b200 import qtip
from paper_2406_11235_b200.layer import QTIPLinear
m, n = int(sys.argv[1]), int(sys.argv[2])
lib = qtip.load()
lib.qtip_internal_set_cta_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
NL = 3
layers = [QTIPLinear(m, n).load_tiles(synth.random_tiles(m, n, 2, seed=i), synth.random_sign_bytes(m, 1),
                                      synth.random_sign_bytes(n, 2)) for i in range(NL)]
x = torch.from_numpy(synth.random_x(1, n, seed=3)).cuda()
y = torch.empty((1, m), device="cuda")
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in layers]
for pdl in (0, 1):
    qtip.set_pdl(bool(pdl))
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    for l in layers:
        l.forward(x, out=y)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for l, (a, b) in zip(layers, ev):
                qtip.profile_events(a, b)
                l.forward(x, out=y)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    CAP = 100000
    buf = torch.zeros(1 + 8 * CAP, dtype=torch.int64, device="cuda")
    lib.qtip_internal_set_cta_trace(buf.data_ptr(), CAP)
    g.replay()
    torch.cuda.synchronize()
    lib.qtip_internal_set_cta_trace(None, 0)
    evt = [a.elapsed_time(b) * 1e3 for a, b in ev]
    b_ = buf.cpu().numpy()
    cnt = int(b_[0])
    r = b_[1:1 + 8 * cnt].reshape(cnt, 8)
    tag = r[:, 0] & 0xFF
    gm = r[(tag == 3) | (tag == 4)]
    gm = gm[np.argsort(gm[:, 3])]
    cuts = np.where(np.diff(gm[:, 3]) > 2000)[0] + 1
    spans = [((p[:, 5].max() - p[:, 3].min()) / 1e3, (p[:, 5].max() - p[:, 4].min()) / 1e3) for p in np.split(gm, cuts)]
    print(f"{m}x{n} pdl={pdl}: events us {np.round(evt, 2)}  trace entry->exit / release->exit {np.round(spans, 2).tolist()}")
