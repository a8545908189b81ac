"""Debug aid: GEMV-kernel time (CUDA events around the kernel) vs cells per CTA."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2406_11235_b200 import qtip
from paper_2406_11235_b200.layer import QTIPLinear
qtip.load()
code = sys.argv[1] if len(sys.argv) > 1 else "3inst"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
impl = int(sys.argv[3]) if len(sys.argv) > 3 else 0
qtip.set_matvec_impl(impl)
fused = int(sys.argv[4]) if len(sys.argv) > 4 else 1
qtip.load().qtip_internal_set_knob(1, fused)
qtip.set_pdl(False)                   # isolate the GEMV kernel in the event timing
n = 4096
for m in [128, 1024, 4736, 9472, 18944, 37888]:
    lay = QTIPLinear(m, n, code=code, k=k).load_tiles(synth.random_tiles(m, n, k), synth.random_sign_bytes(m, 1),
                                                      synth.random_sign_bytes(n, 2), lut=synth.gaussian_lut(9))
    x = torch.from_numpy(synth.random_x(1, n)).cuda()
    for _ in range(3): lay(x, flags=1)
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        qtip.profile_events(a, b)
        lay(x, flags=1)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    units = (m // 128) * (n // 128)
    t = float(np.median(ts))
    print(f"impl={impl} fused={fused} {code} k={k} m={m:6d} units={units:5d} per_cta={units/148:6.2f} gemv_us={t:8.2f} GB/s={m*n*k/8/t/1e3:8.1f}", flush=True)
