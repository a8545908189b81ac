"""Quick GPU probe of the tcgen05 GEMV vs the oracle on a few small shapes (debug aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from oracle import gemv
from paper_2406_11235_b200 import qtip
from paper_2406_11235_b200.layer import QTIPLinear

qtip.load()
for code, k, m, n, B in [("3inst", 2, 128, 128, 1), ("3inst", 2, 256, 384, 1), ("1mad", 2, 256, 256, 2),
                         ("hyb", 4, 256, 256, 1), ("hyb", 3, 256, 256, 3), ("3inst", 2, 384, 768, 16)]:
    tiles = synth.random_tiles(m, n, k, seed=3)
    lut = synth.gaussian_lut(9) if code == "hyb" else None
    lay = QTIPLinear(m, n, code=code, k=k).load_tiles(tiles, synth.random_sign_bytes(m, 1), synth.random_sign_bytes(n, 2), lut=lut)
    x = synth.random_x(B, n, seed=5)
    Wt = gemv.dense_decode(tiles, gemv.Params(k=k, V=2 if code == "hyb" else 1, code=code, lut=lut))
    ref = gemv.matvec(Wt, x, rht_in=False, rht_out=False)
    for impl in (1, 2):
        qtip.set_matvec_impl(impl)
        t = time.time()
        y = lay(torch.from_numpy(x).cuda(), flags=0).cpu().numpy()
        err = np.linalg.norm(y - ref) / np.linalg.norm(ref)
        print(code, k, m, n, B, "impl", impl, "rel", f"{err:.3e}", f"{time.time()-t:.2f}s", flush=True)
