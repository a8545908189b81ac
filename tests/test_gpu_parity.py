"""GPU parity: libqtip (sm_100a, through the C ABI) vs the CPU oracle on identical seeded inputs.

Bars (BASELINE.json north_star): decoded weights bit-exact; matvec relative L2 <= 1e-3 against
the float64 oracle (fp32 accumulation, fp16 activations on the tensor-core path).
"""
import numpy as np
import pytest
import torch

import synth
from oracle import codes, gemv, rht, trellis, viterbi

pytestmark = pytest.mark.gpu

MATVEC_TOL = 1e-3


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def lut_for(code, seed=4000):
    return synth.gaussian_lut(9, seed) if code == "hyb" else None


def make_layer(q, m, n, code, k, tiles, lut=None, seed=0, scale=1.0):
    from paper_2406_11235_b200.layer import QTIPLinear
    layer = QTIPLinear(m, n, code=code, k=k)
    layer.load_tiles(tiles, synth.random_sign_bytes(m, 3001 + seed), synth.random_sign_bytes(n, 3000 + seed),
                     scale=scale, lut=lut)
    return layer


CASES = [("3inst", 2), ("1mad", 2), ("hyb", 4), ("hyb", 3), ("hyb", 2), ("3inst", 3), ("1mad", 4), ("3inst", 1)]


@pytest.mark.parametrize("code,k", CASES)
@pytest.mark.parametrize("m,n", [(256, 256), (272, 304), (128, 512)])
def test_decode_bit_exact(cuda_lib, code, k, m, n):
    tiles = synth.random_tiles(m, n, k, seed=1000 + k * 7 + m)
    lut = lut_for(code)
    layer = make_layer(cuda_lib, m, n, code, k, tiles, lut)
    got = layer.decode().cpu().numpy().view(np.uint16)
    p = gemv.Params(k=k, V=2 if code == "hyb" else 1, code=code, lut=lut)
    ref = gemv.dense_decode(tiles, p).astype(np.float16).view(np.uint16)
    assert np.array_equal(got, ref)
    got32 = layer.decode(out_f32=True).cpu().numpy()
    assert np.array_equal(got32, ref.view(np.float16).astype(np.float32))


def test_decode_kmeans_lut_and_two_sign(cuda_lib):
    m, n = 256, 256
    lut = codes.kmeans_lut(9, seed=4000, n_samples=1 << 15, iters=8)
    tiles = synth.random_tiles(m, n, 4, seed=77)
    for two in (False, True):
        from paper_2406_11235_b200.layer import QTIPLinear
        layer = QTIPLinear(m, n, code="hyb", k=4, two_sign=two)
        layer.load_tiles(tiles, synth.random_sign_bytes(m, 1), synth.random_sign_bytes(n, 2), lut=lut)
        got = layer.decode().cpu().numpy().view(np.uint16)
        ref = gemv.dense_decode(tiles, gemv.Params(k=4, V=2, code="hyb", lut=lut, two_sign=two))
        assert np.array_equal(got, ref.astype(np.float16).view(np.uint16))


def test_c1_viterbi_quantized_tiles_through_pack_states(cuda_lib):
    """Config C1: 256x256, L=16 k=2 V=1 3INST, tail-biting walks from the oracle's Alg. 4 on
    i.i.d. N(0,1) tiles (P:98 'approximately i.i.d. Gaussian'), packed from state walks."""
    m = n = 256
    tab = codes.code_table("3inst", 16)
    sd = tab.std()
    S = synth.gaussian_source((m // 16) * (n // 16), 256, seed=5000)
    states, cost = viterbi.tailbite_encode_batch(S, 16, 2, 1, tab / sd)
    assert (cost / 256).mean() < 0.075                          # ~Table 1 quality
    from paper_2406_11235_b200 import qtip
    from paper_2406_11235_b200.layer import QTIPLinear
    layer = QTIPLinear(m, n, code="3inst", k=2)
    qtip.qtip_pack_states(layer.p, m, n, states.reshape(m // 16, n // 16, 256), layer.packed)
    got = layer.decode().cpu().numpy().view(np.uint16)
    # the oracle's own reconstruction of the same walks
    ref = np.zeros((m, n), dtype=np.uint16)
    vals = codes.decode_3inst(states.astype(np.uint64)).reshape(m // 16, n // 16, 16, 16)
    ref[:] = vals.transpose(0, 2, 1, 3).reshape(m, n)
    assert np.array_equal(got, ref)
    # the decoded tiles approximate the Gaussian source (times the std normaliser)
    src = S.reshape(m // 16, n // 16, 16, 16).transpose(0, 2, 1, 3).reshape(m, n)
    err = ((codes.f16_to_f64(got) / sd - src) ** 2).mean()
    assert err < 0.08
    # a broken walk is rejected
    bad = states.copy()
    bad[3, 10] ^= 0x8000
    with pytest.raises(qtip.QtipError):
        qtip.qtip_pack_states(layer.p, m, n, bad.reshape(m // 16, n // 16, 256), layer.packed)


@pytest.mark.parametrize("n", [256, 4096, 8192, 11008, 28672, 12 * 16, 28 * 8, 20 * 256])
@pytest.mark.parametrize("B", [1, 3, 8, 16])  # 8, 16: the batched plans (rows of D per CTA up to 16)
def test_rht_matches_oracle(cuda_lib, n, B):
    from paper_2406_11235_b200 import qtip
    x = synth.random_x(B, n, seed=2000 + n)
    s = synth.random_sign_bytes(n, 3000)
    dx = torch.from_numpy(x).cuda()
    ds = torch.from_numpy(s).cuda()
    out = torch.empty_like(dx)
    qtip.qtip_rht(n, B, ds, dx, out, inverse=False)
    ref = rht.rht_forward(x, s, n)
    assert rel_l2(out.cpu().numpy(), ref) < 1e-6
    back = torch.empty_like(dx)
    qtip.qtip_rht(n, B, ds, out, back, inverse=True)
    assert rel_l2(back.cpu().numpy(), rht.rht_inverse(out.cpu().numpy().astype(np.float64), s, n)) < 1e-6
    assert rel_l2(back.cpu().numpy(), x) < 1e-5


def _oracle_matvec(tiles, code, k, lut, m, n, x, seed, scale, flags=3, rows=None):
    p = gemv.Params(k=k, V=2 if code == "hyb" else 1, code=code, lut=lut)
    Wt = gemv.dense_decode(tiles, p)
    return gemv.matvec(Wt, x.astype(np.float64), synth.random_sign_bytes(n, 3000 + seed),
                       synth.random_sign_bytes(m, 3001 + seed), scale=scale, rht_in=bool(flags & 1),
                       rht_out=bool(flags & 2), rows=rows)


IMPLS = [1, 2, 3, 4, 5, 6, 7]  # CUDA-core reference, tcgen05 (A in TMEM), register-fed mma.sync, row-tile mma.sync,
                               # fused single-launch layer (k_layer.cu), RHT kernels around the persistent k_layer GEMV,
                               # stream-K tcgen05 GEMV (k_umma.cu, the auto default)


@pytest.mark.parametrize("impl", IMPLS)
@pytest.mark.parametrize("code,k", CASES)
@pytest.mark.parametrize("B", [1, 4, 16])
def test_matvec_small(cuda_lib, impl, code, k, B):
    if impl != 1 and k == 1:
        pytest.skip("tensor-core kernels cover k = 2..4")
    if impl in (4, 5, 6) and B > 4:
        pytest.skip("row-tile and fused layer kernels cover batch 1..4")
    m, n = 384, 768                                          # 3 row blocks x 6 cells
    tiles = synth.random_tiles(m, n, k, seed=11 + k)
    lut = lut_for(code)
    layer = make_layer(cuda_lib, m, n, code, k, tiles, lut, seed=1, scale=0.37)
    x = synth.random_x(B, n, seed=2000 + B)
    cuda_lib.set_matvec_impl(impl)
    try:
        y = layer(torch.from_numpy(x).cuda()).cpu().numpy()
    finally:
        cuda_lib.set_matvec_impl(0)
    ref = _oracle_matvec(tiles, code, k, lut, m, n, x, 1, 0.37)
    tol = 1e-5 if impl == 1 else MATVEC_TOL
    assert rel_l2(y, ref) <= tol


@pytest.mark.parametrize("impl", IMPLS)
def test_matvec_ragged_shapes_and_flags(cuda_lib, impl):
    m, n = 272, 336                                          # partial row block and K-chunk (padding)
    code, k = "3inst", 2
    tiles = synth.random_tiles(m, n, k, seed=5)
    layer = make_layer(cuda_lib, m, n, code, k, tiles, None, seed=2, scale=1.5)
    x = synth.random_x(2, n, seed=9)
    cuda_lib.set_matvec_impl(impl)
    try:
        for flags in (0, 1, 2, 3):
            y = layer(torch.from_numpy(x).cuda(), flags=flags).cpu().numpy()
            ref = _oracle_matvec(tiles, code, k, None, m, n, x, 2, 1.5, flags=flags)
            assert rel_l2(y, ref) <= (1e-5 if impl == 1 else MATVEC_TOL), flags
    finally:
        cuda_lib.set_matvec_impl(0)


@pytest.mark.parametrize("impl", [1, 2, 3, 4, 5, 6])
def test_row_shards_are_bitwise_slices(cuda_lib, impl):
    """Row sharding does not change per-row arithmetic (fixed K-split): shards == full rows bitwise."""
    m, n = 512, 512
    tiles = synth.random_tiles(m, n, 2, seed=8)
    layer = make_layer(cuda_lib, m, n, "3inst", 2, tiles, None, seed=3)
    x = torch.from_numpy(synth.random_x(3, n, seed=4)).cuda()
    cuda_lib.set_matvec_impl(impl)
    try:
        full = layer(x, flags=1).cpu().numpy()
        parts = [layer(x, flags=1, rows=(r, r + 128)).cpu().numpy() for r in range(0, m, 128)]
    finally:
        cuda_lib.set_matvec_impl(0)
    assert np.array_equal(np.concatenate(parts, axis=1), full)


@pytest.mark.parametrize("impl", [2, 3, 4, 5, 6, 7])
@pytest.mark.parametrize("code,k,m,n", [("3inst", 2, 4096, 4096), ("1mad", 2, 11008, 4096), ("3inst", 2, 4096, 11008),
                                        ("hyb", 4, 4096, 4096), ("3inst", 2, 11008, 11008)])
def test_matvec_full_size_sampled_rows(cuda_lib, impl, code, k, m, n):
    """BASELINE C2/C3 shapes in the bench's launch configuration: rows of scale*W~ x~ sampled and
    recomputed one by one by the oracle (RHT-out off), plus the full RHT-out path against the
    oracle's inverse RHT of the GPU's own y~ (a property that holds at any size)."""
    tiles = synth.random_tiles(m, n, k, seed=1000)
    lut = lut_for(code)
    layer = make_layer(cuda_lib, m, n, code, k, tiles, lut, seed=0, scale=0.5)
    x = synth.random_x(1, n, seed=2000)
    dx = torch.from_numpy(x).cuda()
    cuda_lib.set_matvec_impl(impl)
    try:
        yt = layer(dx, flags=1).cpu().numpy()                # scale * W~ x~
        y = layer(dx).cpu().numpy()
    finally:
        cuda_lib.set_matvec_impl(0)
    rows = np.random.default_rng(0).choice(m, 24, replace=False)
    p = gemv.Params(k=k, V=2 if code == "hyb" else 1, code=code, lut=lut)
    Wr = gemv.decode_rows(tiles, p, rows)
    xt = rht.rht_forward(x.astype(np.float64), synth.random_sign_bytes(n, 3000), n)
    ref = 0.5 * (xt @ Wr.T)
    assert rel_l2(yt[:, rows], ref) <= MATVEC_TOL
    ref_y = rht.rht_inverse(yt.astype(np.float64), synth.random_sign_bytes(m, 3001), m)
    assert rel_l2(y, ref_y) <= 1e-5


@pytest.mark.parametrize("code,k", [("3inst", 2), ("hyb", 3), ("1mad", 4)])
@pytest.mark.parametrize("m,n,B", [(688, 688, 1), (448, 896, 2), (896, 448, 4), (4096, 688, 1), (688, 8192, 3),
                                   (16, 32, 1), (32, 16, 2), (176, 144, 1)])
def test_fused_layer_shapes(cuda_lib, code, k, m, n, B):
    """The single-launch layer kernel (impl 5) on Paley (b > 1: dense H_b slices + grid barrier)
    and power-of-two sides, tiny layers (fewer units than CTAs), every batch width it supports."""
    tiles = synth.random_tiles(m, n, k, seed=50 + m + n)
    lut = lut_for(code)
    layer = make_layer(cuda_lib, m, n, code, k, tiles, lut, seed=5, scale=0.8)
    x = synth.random_x(B, n, seed=60 + n)
    cuda_lib.set_matvec_impl(5)
    try:
        ys = [layer(torch.from_numpy(x).cuda(), flags=f).cpu().numpy() for f in (3, 1, 2, 0)]
        again = layer(torch.from_numpy(x).cuda()).cpu().numpy()
    finally:
        cuda_lib.set_matvec_impl(0)
    for f, y in zip((3, 1, 2, 0), ys):
        ref = _oracle_matvec(tiles, code, k, lut, m, n, x, 5, 0.8, flags=f)
        assert rel_l2(y, ref) <= MATVEC_TOL, f
    assert np.array_equal(again, ys[0])                      # barrier epochs carry over between calls


def test_fused_layer_matches_split_path_rows(cuda_lib):
    """impl 5 computes the same rows of scale*W~x~ as the row-tile kernel up to fp32 association."""
    m, n = 1024, 4096
    tiles = synth.random_tiles(m, n, 2, seed=71)
    layer = make_layer(cuda_lib, m, n, "3inst", 2, tiles, None, seed=6)
    x = torch.from_numpy(synth.random_x(1, n, seed=72)).cuda()
    outs = {}
    for impl in (4, 5):
        cuda_lib.set_matvec_impl(impl)
        try:
            outs[impl] = layer(x, flags=1).cpu().numpy()
        finally:
            cuda_lib.set_matvec_impl(0)
    assert rel_l2(outs[5], outs[4]) < 1e-5


def test_matvec_deterministic(cuda_lib):
    m, n = 1024, 2048
    tiles = synth.random_tiles(m, n, 2, seed=1)
    layer = make_layer(cuda_lib, m, n, "3inst", 2, tiles)
    x = torch.from_numpy(synth.random_x(1, n)).cuda()
    a = layer(x).cpu().numpy()
    for _ in range(3):
        assert np.array_equal(layer(x).cpu().numpy(), a)


def test_launch_counter_counts_kernels(cuda_lib):
    m, n = 256, 256
    layer = make_layer(cuda_lib, m, n, "3inst", 2, synth.random_tiles(m, n, 2))
    x = torch.from_numpy(synth.random_x(1, n)).cuda()
    c0 = cuda_lib.launch_count()
    layer(x)
    torch.cuda.synchronize()
    assert cuda_lib.launch_count() > c0


@pytest.mark.parametrize("B", [1, 3])
def test_sharded_layer_world1_nccl_vs_oracle(cuda_lib, B):
    """ShardedQTIPLinear through a real NCCL process group (world size 1 on this GPU): the
    all-gather + replicated RHT-out path against the float64 oracle, and against the unsharded layer."""
    import socket
    import torch.distributed as dist
    from paper_2406_11235_b200.sharded import ShardedQTIPLinear
    m, n = 640, 512
    tiles = synth.random_tiles(m, n, 2, seed=31)
    full = make_layer(cuda_lib, m, n, "3inst", 2, tiles, None, seed=4, scale=0.5)
    xh = synth.random_x(B, n, seed=32)
    x = torch.from_numpy(xh).cuda()
    created = False
    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
        created = True
    try:
        sh = ShardedQTIPLinear(m, n, 0, 1, code="3inst", k=2).load_tiles(
            tiles, synth.random_sign_bytes(m, 3001 + 4), synth.random_sign_bytes(n, 3000 + 4), scale=0.5)
        y_sh = sh(x).cpu().numpy()
    finally:
        if created:
            dist.destroy_process_group()
    ref = _oracle_matvec(tiles, "3inst", 2, None, m, n, xh, 4, 0.5)
    assert rel_l2(y_sh, ref) <= MATVEC_TOL
    assert rel_l2(y_sh, full(x).cpu().numpy()) <= 1e-6


def _two_rank_worker(rank, port, m, n, B, code, k, q):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=2, device_id=torch.device("cuda", rank))
    try:
        from paper_2406_11235_b200 import qtip
        from paper_2406_11235_b200.sharded import ShardedQTIPLinear
        qtip.load()
        lut = synth.gaussian_lut(9) if code == "hyb" else None
        tiles = synth.random_tiles(m, n, k, seed=41)
        sh = ShardedQTIPLinear(m, n, rank, 2, code=code, k=k, device=torch.device("cuda", rank)).load_tiles(
            tiles, synth.random_sign_bytes(m, 43), synth.random_sign_bytes(n, 42), scale=0.75, lut=lut)
        x = torch.from_numpy(synth.random_x(B, n, seed=44)).cuda(rank)
        q.put((rank, sh(x).cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("code,k,m,n,B", [("3inst", 2, 640, 512, 1), ("hyb", 4, 1152, 256, 3)])
def test_sharded_layer_two_ranks_nccl_vs_oracle(cuda_lib, code, k, m, n, B):
    """Two ranks (one GPU each) over NCCL: uneven row shards (5 and 9 row blocks -> 3+2, 5+4), the
    all-gather with reorder, the replicated RHT-out; every rank's y against the float64 oracle.
    Skipped when fewer than two GPUs are visible (the round's pool gives one GPU per call)."""
    import socket
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_two_rank_worker, args=(r, port, m, n, B, code, k, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    lut = synth.gaussian_lut(9) if code == "hyb" else None
    tiles = synth.random_tiles(m, n, k, seed=41)
    p = gemv.Params(k=k, V=2 if code == "hyb" else 1, code=code, lut=lut)
    ref = gemv.matvec(gemv.dense_decode(tiles, p), synth.random_x(B, n, seed=44).astype(np.float64),
                      synth.random_sign_bytes(n, 42), synth.random_sign_bytes(m, 43), scale=0.75)
    for rank, y in res:
        assert rel_l2(y, ref) <= MATVEC_TOL, rank


@pytest.mark.parametrize("k", [2, 3, 4])
@pytest.mark.parametrize("impl", [0, 5, 6])
def test_hyb_two_sign_matvec(cuda_lib, k, impl):
    """HYB two-sign variant (bit 31 of x^2 + x also flips the first entry) through the
    shared-memory LUT fast path: matvec within 1e-3 of the float64 oracle."""
    from paper_2406_11235_b200.layer import QTIPLinear
    m, n = 384, 768
    tiles = synth.random_tiles(m, n, k, seed=90 + k)
    lut = lut_for("hyb")
    layer = QTIPLinear(m, n, code="hyb", k=k, two_sign=True)
    layer.load_tiles(tiles, synth.random_sign_bytes(m, 3001 + 7), synth.random_sign_bytes(n, 3000 + 7), scale=0.6, lut=lut)
    x = synth.random_x(1, n, seed=91)
    cuda_lib.set_matvec_impl(impl)
    try:
        y = layer(torch.from_numpy(x).cuda()).cpu().numpy()
    finally:
        cuda_lib.set_matvec_impl(0)
    p = gemv.Params(k=k, V=2, code="hyb", lut=lut, two_sign=True)
    ref = gemv.matvec(gemv.dense_decode(tiles, p), x.astype(np.float64), synth.random_sign_bytes(n, 3000 + 7),
                      synth.random_sign_bytes(m, 3001 + 7), scale=0.6)
    assert rel_l2(y, ref) <= MATVEC_TOL


def test_empty_batch_is_a_no_op(cuda_lib):
    """B = 0: an empty (0, m) result and no kernel launch (the ABI itself refuses B < 1)."""
    layer = make_layer(cuda_lib, 256, 256, "3inst", 2, synth.random_tiles(256, 256, 2, seed=3))
    c0 = cuda_lib.launch_count()
    y = layer(torch.empty((0, 256), dtype=torch.float32, device="cuda"))
    assert tuple(y.shape) == (0, 256) and cuda_lib.launch_count() == c0


@pytest.mark.parametrize("impl", IMPLS)
def test_zero_input_gives_exact_zero(cuda_lib, impl):
    """x = 0: every path returns exact zeros (no NaN from the fp16 x~ or the scale)."""
    m, n = 384, 768
    layer = make_layer(cuda_lib, m, n, "hyb", 3, synth.random_tiles(m, n, 3, seed=4), lut_for("hyb"), scale=3.0)
    cuda_lib.set_matvec_impl(impl)
    try:
        y = layer(torch.zeros((2, n), dtype=torch.float32, device="cuda")).cpu().numpy()
    finally:
        cuda_lib.set_matvec_impl(0)
    assert np.array_equal(y, np.zeros_like(y))


@pytest.mark.parametrize("impl", IMPLS)
@pytest.mark.parametrize("m,n", [(16, 16), (16, 48), (48, 16)])
def test_smallest_layers(cuda_lib, impl, m, n):
    """One-tile-high / one-tile-wide layers (less than one 128-row block, one K-chunk)."""
    tiles = synth.random_tiles(m, n, 2, seed=m + n)
    layer = make_layer(cuda_lib, m, n, "3inst", 2, tiles, None, seed=6, scale=0.5)
    x = synth.random_x(1, n, seed=7)
    cuda_lib.set_matvec_impl(impl)
    try:
        y = layer(torch.from_numpy(x).cuda()).cpu().numpy()
    finally:
        cuda_lib.set_matvec_impl(0)
    ref = _oracle_matvec(tiles, "3inst", 2, None, m, n, x, 6, 0.5)
    assert rel_l2(y, ref) <= (1e-5 if impl == 1 else MATVEC_TOL)


@pytest.mark.parametrize("code,k", [("3inst", 2), ("hyb", 4)])
def test_maximum_batch(cuda_lib, code, k):
    """B = 64, the largest batch the ABI accepts (auto kernel choice)."""
    m, n = 256, 512
    tiles = synth.random_tiles(m, n, k, seed=21)
    lut = lut_for(code)
    layer = make_layer(cuda_lib, m, n, code, k, tiles, lut, seed=8)
    x = synth.random_x(64, n, seed=22)
    y = layer(torch.from_numpy(x).cuda()).cpu().numpy()
    ref = _oracle_matvec(tiles, code, k, lut, m, n, x, 8, 1.0)
    assert rel_l2(y, ref) <= MATVEC_TOL


@pytest.mark.parametrize("code,k,G,m,n,B,grouped", [("3inst", 2, 3, 1024, 512, 1, True), ("hyb", 4, 2, 1280, 256, 2, True),
                                                    ("1mad", 3, 4, 688, 256, 4, True), ("3inst", 2, 3, 256, 256, 1, False),
                                                    ("hyb", 4, 2, 11008, 4096, 4, None)])
def test_grouped_impl6_equals_per_layer_calls(cuda_lib, code, k, G, m, n, B, grouped):
    """The persistent-kernel grouping (impl 6): qtip_matvec_group == G qtip_matvec calls, bit for bit,
    for every flag combination, when the group ran as one launch (one RHT-in + one GEMV (+ one RHT-out));
    else (256 rows: too few tile rows per CTA; 11008 x 4096 at B = 4: the plan does not fit shared
    memory) G per-layer impl-6-or-fallback calls."""
    from paper_2406_11235_b200.layer import forward_group
    lut = lut_for(code)
    tiles = [synth.random_tiles(m, n, k, seed=50 + g) for g in range(G)]
    layers = [make_layer(cuda_lib, m, n, code, k, tiles[g], lut, seed=20 + g, scale=0.5 + g) for g in range(G)]
    x = torch.from_numpy(synth.random_x(B, n, seed=77)).cuda()
    cuda_lib.set_matvec_impl(6)
    try:
        for flags in (1, 3, 0, 2):
            c0 = cuda_lib.launch_count()
            outs = [o.cpu().numpy() for o in forward_group(layers, x, flags=flags)]
            launches = cuda_lib.launch_count() - c0
            ran_grouped = launches == 2 + bool(flags & 2)
            if flags & 1 and grouped is not None:
                assert ran_grouped == grouped, (flags, launches)
            if ran_grouped and flags & 1:
                ref = [l(x, flags=flags).cpu().numpy() for l in layers]
                for g in range(G):
                    assert np.array_equal(outs[g], ref[g]), (flags, g)
            if flags == 3 and m * n <= 1 << 20:
                want = _oracle_matvec(tiles[0], code, k, lut, m, n, x.cpu().numpy(), 20, 0.5)
                assert rel_l2(outs[0], want) <= MATVEC_TOL
    except cuda_lib.QtipError as e:
        assert not grouped, e                                # impl 6 refuses the ungrouped shapes
    finally:
        cuda_lib.set_matvec_impl(0)


@pytest.mark.parametrize("code,k,G,m,n,B", [("3inst", 2, 3, 1024, 512, 1), ("hyb", 4, 2, 1280, 256, 2),
                                            ("1mad", 3, 4, 688, 256, 4), ("3inst", 2, 3, 256, 256, 1),
                                            ("hyb", 3, 2, 1024, 8192, 1), ("3inst", 2, 2, 384, 768, 16)])
def test_grouped_matvec_against_oracle(cuda_lib, code, k, G, m, n, B):
    """qtip_matvec_group as the bench runs it (auto: one grouped RHT-in, one stream-K tcgen05 launch
    over the G layers' cells, one grouped RHT-out / segment reduction): every member, every row,
    every flag combination against the float64 oracle."""
    from paper_2406_11235_b200.layer import forward_group
    lut = lut_for(code)
    tiles = [synth.random_tiles(m, n, k, seed=50 + g) for g in range(G)]
    layers = [make_layer(cuda_lib, m, n, code, k, tiles[g], lut, seed=20 + g, scale=0.5 + g) for g in range(G)]
    xh = synth.random_x(B, n, seed=77)
    x = torch.from_numpy(xh).cuda()
    p = gemv.Params(k=k, V=2 if code == "hyb" else 1, code=code, lut=lut)
    W = [gemv.dense_decode(tiles[g], p) for g in range(G)]
    for flags in (3, 1, 0, 2):
        outs = [o.cpu().numpy() for o in forward_group(layers, x, flags=flags)]
        for g in range(G):
            want = gemv.matvec(W[g], xh.astype(np.float64), synth.random_sign_bytes(n, 3000 + 20 + g),
                               synth.random_sign_bytes(m, 3001 + 20 + g), scale=0.5 + g, rht_in=bool(flags & 1),
                               rht_out=bool(flags & 2))
            assert rel_l2(outs[g], want) <= MATVEC_TOL, (flags, g)


def test_grouped_two_sign_hyb_and_distinct_luts(cuda_lib):
    """Grouped launch with HYB two-sign and a different LUT per member: each member
    against its own per-layer impl 6 call (bitwise) and the oracle."""
    from paper_2406_11235_b200.layer import QTIPLinear, forward_group
    m, n, k, G = 1280, 512, 3, 2
    luts = [synth.gaussian_lut(9, 4100 + g) for g in range(G)]
    tiles = [synth.random_tiles(m, n, k, seed=95 + g) for g in range(G)]
    layers = []
    for g in range(G):
        l = QTIPLinear(m, n, code="hyb", k=k, two_sign=True)
        l.load_tiles(tiles[g], synth.random_sign_bytes(m, 3101 + g), synth.random_sign_bytes(n, 3100 + g),
                     scale=0.7 + g, lut=luts[g])
        layers.append(l)
    x = torch.from_numpy(synth.random_x(1, n, seed=96)).cuda()
    c0 = cuda_lib.launch_count()
    outs = [o.cpu().numpy() for o in forward_group(layers, x)]
    assert cuda_lib.launch_count() - c0 == 3                     # grouped RHT-in, GEMV, RHT-out
    cuda_lib.set_matvec_impl(6)
    try:
        ref = [l(x).cpu().numpy() for l in layers]
    finally:
        cuda_lib.set_matvec_impl(0)
    for g in range(G):
        assert np.array_equal(outs[g], ref[g]), g
        p = gemv.Params(k=k, V=2, code="hyb", lut=luts[g], two_sign=True)
        want = gemv.matvec(gemv.dense_decode(tiles[g], p), x.cpu().numpy().astype(np.float64),
                           synth.random_sign_bytes(n, 3100 + g), synth.random_sign_bytes(m, 3101 + g), scale=0.7 + g)
        assert rel_l2(outs[g], want) <= MATVEC_TOL
