"""Debug aid: timeline of the tcgen05 GEMV's CTA 0 (clock64 per hand-off)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2406_11235_b200 import qtip
from paper_2406_11235_b200.layer import QTIPLinear
lib = qtip.load()
qtip.set_matvec_impl(int(os.environ.get("QTIP_IMPL", "0")))
m, n = int(sys.argv[1]) if len(sys.argv) > 1 else 11008, 4096
lay = QTIPLinear(m, n).load_tiles(synth.random_tiles(m, n, 2), synth.random_sign_bytes(m, 1), synth.random_sign_bytes(n, 2))
x = torch.from_numpy(synth.random_x(1, n)).cuda()
for _ in range(3): lay(x)
tr = torch.zeros(256 * 8, dtype=torch.int64, device="cuda")
lib.qtip_internal_set_trace.argtypes = [ctypes.c_void_p]
lib.qtip_internal_set_trace(ctypes.c_void_p(tr.data_ptr()))
lay(x); torch.cuda.synchronize()
lib.qtip_internal_set_trace(None)
t = tr.cpu().numpy().reshape(256, 8).astype(np.int64)
ns = t[255]
print("CTA0 globaltimer ns: setup=%d first-decoder-done=%d exit=%d" % (ns[1] - ns[0], ns[2] - ns[0], ns[3] - ns[0]))
t[255] = 0
t0 = t[t > 0].min()
names = ["wait0", "waitok", "decoded", "barok", "issued", "epi_done", "strm0", "strmok"]
for g in range(4):
    for hc in range(16):
        row = t[g * 64 + hc]
        if row.max() == 0: continue
        print(f"g{g} hc{hc:2d} " + " ".join(f"{nm}={(v - t0) if v else -1:7d}" for nm, v in zip(names, row)))
