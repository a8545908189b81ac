"""CPU-side checks of the C-ABI library: it builds/loads, exports every symbol declared in
include/qtip.h, and its host-only logic (params, sizes, Hadamard factorisation, Paley
tables, error codes) behaves as documented.  No device compute runs here."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2406_11235_b200 import build, qtip

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return qtip.load()


def header_functions():
    src = open(os.path.join(ROOT, "include", "qtip.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(qtip_[a-z_0-9]+)\s*\(", src)
    return sorted(set(names))


def test_exports_every_declared_symbol(lib):
    names = header_functions()
    assert len(names) >= 15
    for nm in names:
        assert hasattr(lib, nm), nm
    assert set(qtip.EXPORTS) <= set(names)


def test_params_defaults_follow_the_paper(lib):
    p = qtip.params_default("3inst", 2)
    assert (p.L, p.k, p.V, p.lcg_a, p.lcg_b, p.m_fp16, p.Q) == (16, 2, 1, 89226354, 64248484, 0x3B60, 9)
    p = qtip.params_default("1mad", 2)
    assert (p.lcg_a, p.lcg_b, p.V) == (34038481, 76625530, 1)
    p = qtip.params_default("hyb", 4)
    assert (p.V, p.Q, p.tail_biting, p.Tx, p.Ty) == (2, 9, 1, 16, 16)
    assert qtip.params_check(p) == 0


def test_params_check_errors(lib):
    p = qtip.params_default("3inst", 2)
    p.V = 2
    assert qtip.params_check(p) == -1
    p = qtip.params_default("hyb", 4)
    p.V = 1
    assert qtip.params_check(p) == 0             # HYB with a 1-D codebook, k_variant.cu
    p.V = 3
    assert qtip.params_check(p) == -1
    p = qtip.params_default("3inst", 2)
    p.L = 12
    assert qtip.params_check(p) == -5            # valid QTIP, unsupported on the device path
    p = qtip.params_default("3inst", 2)
    p.tail_biting = 0
    assert qtip.params_check(p) == -5
    p = qtip.params_default("3inst", 5)
    assert qtip.params_check(p) == -1
    assert lib.qtip_params_check(None) == -1


def test_packed_bytes(lib):
    p = qtip.params_default("3inst", 2)
    assert qtip.packed_bytes(p, 4096, 4096) == 4096 * 4096 * 2 // 8
    assert qtip.packed_bytes(p, 11008, 4096) == 11008 * 4096 * 2 // 8      # 11008 = 86 * 128, no padding
    assert qtip.packed_bytes(p, 4096, 11008) == 4096 * 11008 * 2 // 8      # 11008 = 86 * 128
    assert qtip.packed_bytes(p, 16, 16) == 128 * 128 * 2 // 8               # one padded cell
    assert qtip.packed_bytes(p, 17, 16) == -1
    assert qtip.packed_bytes(qtip.params_default("hyb", 3), 8192, 28672) == 8192 * 28672 * 3 // 8


def test_hadamard_factorisation_matches_reading(lib):
    assert qtip.hadamard_order(4096) == (1, 12)
    assert qtip.hadamard_order(11008) == (344, 5)
    assert qtip.hadamard_order(28672) == (28, 10)
    assert qtip.hadamard_order(5120) == (20, 8)
    with pytest.raises(qtip.QtipError):
        qtip.hadamard_order(105)


@pytest.mark.parametrize("b", [4, 12, 20, 28, 108, 344])
def test_library_paley_tables_are_hadamard(lib, b):
    H = qtip.paley_host(b).astype(np.int64)
    assert (H @ H.T == b * np.eye(b, dtype=np.int64)).all()
    assert (H + H.T == 2 * np.eye(b, dtype=np.int64)).all()


def test_status_strings(lib):
    assert lib.qtip_status_string(0) == b"QTIP_OK"
    assert lib.qtip_status_string(-3) == b"QTIP_ERR_INVALID_PATH"


def test_host_validation_before_any_launch(lib):
    """Calls with invalid arguments return an error without touching the device."""
    p = qtip.params_default("3inst", 2)
    vp = ctypes.c_void_p
    assert lib.qtip_decode(ctypes.byref(p), 17, 16, vp(16), None, 0, vp(16), None) == -2
    assert lib.qtip_decode(ctypes.byref(p), 16, 16, None, None, 0, vp(16), None) == -1
    assert lib.qtip_decode(ctypes.byref(p), 16, 16, vp(8), None, 0, vp(16), None) == -4
    assert lib.qtip_rht(105, 1, vp(16), vp(16), vp(32), 0, None) == -2
    assert lib.qtip_rht(256, 1, vp(16), vp(16), vp(16), 0, None) == -1      # in-place refused
    ws = 1 << 20
    # partial row range with RHT_OUT is refused
    assert lib.qtip_matvec(ctypes.byref(p), 256, 256, 1, vp(256), None, vp(256), vp(256), ctypes.c_float(1.0),
                           vp(256), vp(256), 128, 256, 3, vp(256), ws, None) == -1
    assert lib.qtip_matvec(ctypes.byref(p), 256, 256, 1, vp(256), None, vp(256), vp(256), ctypes.c_float(1.0),
                           vp(256), vp(256), 64, 256, 0, vp(256), ws, None) == -2
    assert lib.qtip_matvec(ctypes.byref(p), 256, 256, 1, vp(256), None, vp(256), vp(256), ctypes.c_float(1.0),
                           vp(256), vp(256), 0, 256, 3, vp(256), 16, None) == -7
    # qtip_pack_states rejects a non-walk before copying anything
    states = np.zeros((1, 1, 256), dtype=np.uint32)
    states[0, 0, 5] = 0xFFFF
    assert lib.qtip_pack_states(ctypes.byref(p), 16, 16, states.ctypes.data_as(vp), vp(256), None) == -3


def test_degenerate_arguments_are_refused(lib):
    """Empty and out-of-range sizes return a status (include/qtip.h) before any device access;
    the Python layers map an empty batch / no sequences to an empty result without a call."""
    p = qtip.params_default("3inst", 2)
    vp, f1, ws = ctypes.c_void_p, ctypes.c_float(1.0), 1 << 20

    def mv(m=256, n=256, B=1, r0=0, r1=256, flags=3, sn=vp(256), sm=vp(256)):
        return lib.qtip_matvec(ctypes.byref(p), m, n, B, vp(256), None, sn, sm, f1, vp(256), vp(512), r0, r1,
                               flags, vp(256), ws, None)
    assert mv(B=0) == -1 and mv(B=65) == -1                        # batch 1..64
    assert mv(r0=128, r1=128, flags=0) == -2                       # empty row range
    assert mv(m=0, r1=0) == -2 and mv(n=0) == -2 and mv(m=250, r1=250) == -2   # multiples of 16
    assert mv(flags=8) == -1                                       # unknown flag
    assert mv(sn=None) == -1 and mv(sm=None) == -1                 # RHT without its signs
    assert lib.qtip_rht(256, 0, vp(16), vp(16), vp(32), 0, None) == -2
    assert lib.qtip_rht(0, 1, vp(16), vp(16), vp(32), 0, None) == -2
    pv = qtip.params_default("3inst", 2)

    def vt(nseq=1, T=256, pp=pv):
        return lib.qtip_viterbi_tailbite(ctypes.byref(pp), nseq, T, vp(256), None, vp(256), vp(256), vp(256),
                                         1 << 30, None)
    assert vt(nseq=0) == -2 and vt(T=1) == -2 and vt(T=4097) == -2
    ph = qtip.params_default("hyb", 2)
    assert vt(T=255, pp=ph) == -2                                  # V = 2 must divide T
    p1 = qtip.params_default("3inst", 1)
    assert vt(pp=p1) == -5                                         # V = 1 Viterbi: k in {2, 3, 4}
    pq = qtip.params_default("hyb", 2)
    pq.Q = 6
    assert vt(pp=pq) == -5                                         # HYB Viterbi: Q = 9



def test_group_call_validation(lib):
    """qtip_matvec_group refuses bad group sizes, NULL arrays and per-member errors before any launch."""
    p = qtip.params_default("3inst", 2)
    vp = ctypes.c_void_p
    lib.qtip_matvec_group.argtypes = [ctypes.POINTER(qtip.QtipParams), ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp),
                                      ctypes.POINTER(vp), ctypes.POINTER(ctypes.c_float), vp, ctypes.POINTER(vp),
                                      ctypes.c_int, ctypes.POINTER(vp), ctypes.c_size_t, vp]
    lib.qtip_matvec_group.restype = ctypes.c_int
    G = 3
    arr = lambda v: (vp * G)(*([vp(v)] * G))
    sc = (ctypes.c_float * G)(1.0, 1.0, 1.0)
    ws = 1 << 20

    def call(G=3, m=256, n=256, B=1, flags=3, packed=None, sn=None, wsb=ws):
        return lib.qtip_matvec_group(ctypes.byref(p), G, m, n, B, packed or arr(256), None, sn or arr(256), arr(256), sc,
                                     vp(256), arr(512), flags, arr(256), wsb, None)
    assert call(G=0) == -1 and call(G=5) == -1                     # group size 1..4
    assert call(B=0) == -1 and call(m=250) == -2 and call(flags=8) == -1
    assert call(packed=(vp * G)(vp(256), None, vp(256))) == -1   # NULL member buffer
    assert call(packed=arr(8)) == -4                               # misaligned member stream
    assert call(wsb=16) == -7                                      # workspace too small
    assert lib.qtip_matvec_group(ctypes.byref(p), 3, 256, 256, 1, None, None, arr(256), arr(256), sc, vp(256), arr(512),
                                 3, arr(256), ws, None) == -1


def _chain_status(lib, p, layers, B=1, lut=None):
    arr = (qtip.ChainLayer * len(layers))()
    for i, d in enumerate(layers):
        arr[i] = qtip.ChainLayer(0x1000, 0x2000, 0x3000, 1.0, d[0], d[1], 0x4000, d[2], d[3])
    plan = ctypes.c_void_p()
    return lib.qtip_chain_plan_create(ctypes.byref(p), len(layers), arr, B, lut, ctypes.byref(plan))


def test_chain_plan_validation(lib):
    """qtip_chain_plan_create rejects malformed chains on the host, before any device call."""
    p = qtip.params_default("3inst", 2)
    ok_a = (512, 256, 0, -1)
    # stage numbers must start at 0 and grow by one
    assert _chain_status(lib, p, [(512, 256, 1, -1)]) == -1
    assert _chain_status(lib, p, [ok_a, (256, 512, 2, 0)]) == -1
    # stage 0 reads x; later stages read a layer of the previous stage with m == n
    assert _chain_status(lib, p, [(512, 256, 0, 0)]) == -1
    assert _chain_status(lib, p, [ok_a, (256, 256, 1, 0)]) == -2
    assert _chain_status(lib, p, [ok_a, (256, 512, 1, -1)]) == -1
    # a stage shares n and src; at most 4 layers per stage
    assert _chain_status(lib, p, [ok_a, (512, 128, 0, -1)]) == -1
    assert _chain_status(lib, p, [ok_a] * 5) == -5
    # batch 1..16, k 2..4, HYB needs its LUT
    assert _chain_status(lib, p, [ok_a], B=17) == -5
    assert _chain_status(lib, p, [ok_a], B=0) == -5
    assert _chain_status(lib, qtip.params_default("3inst", 1), [ok_a]) == -5
    assert _chain_status(lib, qtip.params_default("hyb", 4), [ok_a]) == -5
    # shapes: positive multiples of 16
    assert _chain_status(lib, p, [(520, 256, 0, -1)]) == -2
    assert _chain_status(lib, p, [(512, 40, 0, -1)]) == -2
    assert lib.qtip_chain_run(None, None, None) == -1
    lib.qtip_chain_plan_destroy(None)
    assert lib.qtip_chain_plan_stages(None) == 0


def test_params_check_code_variants(lib):
    """NEXT-3 variants: the lookup-only code (L <= 16, 16x16 or 32x8 blocks) and HYB with V = 1."""
    p = qtip.params_default("lut", 2)
    assert (p.L, p.V, p.Tx, p.Ty, p.code) == (14, 1, 32, 8, 4)
    assert qtip.params_check(p) == 0
    p.Tx, p.Ty = 16, 16
    assert qtip.params_check(p) == 0
    p.Tx, p.Ty = 64, 4
    assert qtip.params_check(p) == -5
    p.Tx, p.Ty = 32, 16
    assert qtip.params_check(p) == -1                         # T = Tx Ty must be 256
    p = qtip.params_default("lut", 2)
    p.L = 17
    assert qtip.params_check(p) == -5
    p = qtip.params_default("hyb1", 2)
    assert (p.V, p.Q, p.code) == (1, 6, 3) and qtip.params_check(p) == 0
    p.Q = 15
    assert qtip.params_check(p) == -5
    p = qtip.params_default("3inst", 2)
    p.Tx, p.Ty = 32, 8
    assert qtip.params_check(p) == -5                         # 32 x 8 blocks: the LUT code only
    # 32 x 8 blocks need m % 32 == 0
    p = qtip.params_default("lut", 2)
    assert lib.qtip_pack(ctypes.byref(p), 48, 64, np.zeros(64 * 48 // 256 * 64, np.uint8).ctypes.data_as(ctypes.c_void_p),
                         ctypes.c_void_p(16), None) == -2
