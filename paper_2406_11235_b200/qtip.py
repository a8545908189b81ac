"""Thin Python binding of libqtip (include/qtip.h): argument marshalling only.

Every computation runs in libqtip's sm_100a kernels; this module converts torch tensors
(device buffers, current stream) and numpy arrays (host buffers) to the C ABI's plain
pointers and raises on a non-OK status.  It never falls back to a CPU implementation:
if libqtip.so is missing it raises.
"""
import ctypes
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libqtip.so")

QTIP_CODE_1MAD, QTIP_CODE_3INST, QTIP_CODE_HYB, QTIP_CODE_LUT = 1, 2, 3, 4
# "hyb1": HYB with a 1-D codebook (V = 1, Q = 6); "lut": the lookup-only code
# (L = 14, V = 1, T_x x T_y = 32 x 8)
CODES = {"1mad": QTIP_CODE_1MAD, "3inst": QTIP_CODE_3INST, "hyb": QTIP_CODE_HYB, "hyb1": QTIP_CODE_HYB,
         "lut": QTIP_CODE_LUT}
QTIP_RHT_IN, QTIP_RHT_OUT = 1, 2
QTIP_XT_READY = 4          # kernel benchmarking: reuse the x~ already in the workspace
IMPL_AUTO, IMPL_SIMPLE, IMPL_TC, IMPL_MMA = 0, 1, 2, 3

STATUS = {0: "QTIP_OK", -1: "QTIP_ERR_INVALID_PARAMS", -2: "QTIP_ERR_SHAPE", -3: "QTIP_ERR_INVALID_PATH",
          -4: "QTIP_ERR_ALIGNMENT", -5: "QTIP_ERR_UNSUPPORTED", -6: "QTIP_ERR_CUDA", -7: "QTIP_ERR_WORKSPACE"}

EXPORTS = ["qtip_params_default", "qtip_params_check", "qtip_packed_bytes", "qtip_pack", "qtip_pack_states",
           "qtip_decode", "qtip_matvec", "qtip_matvec_group", "qtip_matvec_group_fused", "qtip_matvec_workspace_bytes", "qtip_rht", "qtip_hadamard_order",
           "qtip_set_matvec_impl", "qtip_get_matvec_impl", "qtip_status_string", "qtip_last_error",
           "qtip_launch_count", "qtip_profile_events", "qtip_set_pdl", "qtip_viterbi_workspace_bytes",
           "qtip_viterbi_tailbite", "qtip_chain_plan_create", "qtip_chain_run", "qtip_chain_plan_destroy",
           "qtip_chain_plan_stages", "qtip_quantize_workspace_bytes", "qtip_quantize_matrix"]


class QtipParams(ctypes.Structure):
    _fields_ = [("L", ctypes.c_int32), ("k", ctypes.c_int32), ("V", ctypes.c_int32), ("code", ctypes.c_int32),
                ("Q", ctypes.c_int32), ("tail_biting", ctypes.c_int32), ("Tx", ctypes.c_int32), ("Ty", ctypes.c_int32),
                ("lcg_a", ctypes.c_uint32), ("lcg_b", ctypes.c_uint32), ("m_fp16", ctypes.c_uint32),
                ("hyb_two_sign", ctypes.c_int32)]


class ChainLayer(ctypes.Structure):
    _fields_ = [("d_packed", ctypes.c_void_p), ("d_sign_n", ctypes.c_void_p), ("d_sign_m", ctypes.c_void_p),
                ("scale", ctypes.c_float), ("m", ctypes.c_int64), ("n", ctypes.c_int64), ("d_y", ctypes.c_void_p),
                ("stage", ctypes.c_int32), ("src", ctypes.c_int32)]


class QtipError(RuntimeError):
    def __init__(self, fn, status, detail):
        super().__init__(f"{fn}: {STATUS.get(status, status)}: {detail}")
        self.status = status


_lib = None


def load(path=LIB_PATH):
    """Load libqtip.so (built by paper_2406_11235_b200.build / __graft_entry__.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libqtip.so not found at {path}: run `python -m paper_2406_11235_b200.build` "
                           "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    P = ctypes.POINTER(QtipParams)
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
    lib.qtip_params_default.argtypes = [P, i32, i32]
    lib.qtip_params_default.restype = None
    lib.qtip_params_check.argtypes = [P]
    lib.qtip_params_check.restype = ctypes.c_int
    lib.qtip_packed_bytes.argtypes = [P, i64, i64]
    lib.qtip_packed_bytes.restype = i64
    lib.qtip_pack.argtypes = [P, i64, i64, vp, vp, vp]
    lib.qtip_pack.restype = ctypes.c_int
    lib.qtip_pack_states.argtypes = [P, i64, i64, vp, vp, vp]
    lib.qtip_pack_states.restype = ctypes.c_int
    lib.qtip_decode.argtypes = [P, i64, i64, vp, vp, ctypes.c_int, vp, vp]
    lib.qtip_decode.restype = ctypes.c_int
    lib.qtip_matvec.argtypes = [P, i64, i64, i64, vp, vp, vp, vp, ctypes.c_float, vp, vp, i64, i64, ctypes.c_int,
                                vp, ctypes.c_size_t, vp]
    lib.qtip_matvec.restype = ctypes.c_int
    PP = ctypes.POINTER(vp)
    lib.qtip_matvec_group.argtypes = [P, ctypes.c_int, i64, i64, i64, PP, PP, PP, PP, ctypes.POINTER(ctypes.c_float),
                                      vp, PP, ctypes.c_int, PP, ctypes.c_size_t, vp]
    lib.qtip_matvec_group.restype = ctypes.c_int
    lib.qtip_matvec_group_fused.argtypes = [P, ctypes.c_int, i64, i64, i64]
    lib.qtip_matvec_group_fused.restype = ctypes.c_int
    lib.qtip_matvec_workspace_bytes.argtypes = [P, i64, i64, i64]
    lib.qtip_matvec_workspace_bytes.restype = ctypes.c_size_t
    lib.qtip_rht.argtypes = [i64, i64, vp, vp, vp, ctypes.c_int, vp]
    lib.qtip_rht.restype = ctypes.c_int
    lib.qtip_hadamard_order.argtypes = [i64, ctypes.POINTER(i32), ctypes.POINTER(i32)]
    lib.qtip_hadamard_order.restype = ctypes.c_int
    lib.qtip_viterbi_workspace_bytes.argtypes = [P, i64]
    lib.qtip_viterbi_workspace_bytes.restype = ctypes.c_size_t
    lib.qtip_viterbi_tailbite.argtypes = [P, i64, i64, vp, vp, vp, vp, vp, ctypes.c_size_t, vp]
    lib.qtip_viterbi_tailbite.restype = ctypes.c_int
    lib.qtip_set_matvec_impl.argtypes = [ctypes.c_int]
    lib.qtip_set_matvec_impl.restype = None
    lib.qtip_get_matvec_impl.argtypes = []
    lib.qtip_get_matvec_impl.restype = ctypes.c_int
    lib.qtip_status_string.argtypes = [ctypes.c_int]
    lib.qtip_status_string.restype = ctypes.c_char_p
    lib.qtip_last_error.argtypes = []
    lib.qtip_last_error.restype = ctypes.c_char_p
    lib.qtip_launch_count.argtypes = []
    lib.qtip_launch_count.restype = ctypes.c_uint64
    lib.qtip_profile_events.argtypes = [vp, vp]
    lib.qtip_profile_events.restype = None
    lib.qtip_set_pdl.argtypes = [ctypes.c_int]
    lib.qtip_set_pdl.restype = None
    lib.qtip_quantize_workspace_bytes.argtypes = [P, i64, i64]
    lib.qtip_quantize_workspace_bytes.restype = ctypes.c_size_t
    lib.qtip_quantize_matrix.argtypes = [P, i64, i64, vp, ctypes.c_float, vp, vp, vp, vp, ctypes.c_size_t, vp]
    lib.qtip_quantize_matrix.restype = ctypes.c_int
    lib.qtip_chain_plan_create.argtypes = [P, i32, ctypes.POINTER(ChainLayer), i64, vp, ctypes.POINTER(vp)]
    lib.qtip_chain_plan_create.restype = ctypes.c_int
    lib.qtip_chain_run.argtypes = [vp, vp, vp]
    lib.qtip_chain_run.restype = ctypes.c_int
    lib.qtip_chain_plan_destroy.argtypes = [vp]
    lib.qtip_chain_plan_destroy.restype = None
    lib.qtip_chain_plan_stages.argtypes = [vp]
    lib.qtip_chain_plan_stages.restype = i32
    _lib = lib
    return lib


def _check(fn, st):
    if st != 0:
        raise QtipError(fn, st, load().qtip_last_error().decode())


def _ptr(t):
    """Device pointer of a torch tensor (or None)."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


@dataclass
class Config:
    code: str = "3inst"
    k: int = 2
    two_sign: bool = False

    def params(self):
        p = QtipParams()
        load().qtip_params_default(ctypes.byref(p), CODES[self.code], self.k)
        p.hyb_two_sign = int(self.two_sign)
        if self.code == "hyb1":
            p.V, p.Q = 1, 6
        return p


def params_default(code="3inst", k=2, two_sign=False):
    return Config(code, k, two_sign).params()


def params_check(p):
    return load().qtip_params_check(ctypes.byref(p))


def packed_bytes(p, m, n):
    return load().qtip_packed_bytes(ctypes.byref(p), m, n)


def qtip_pack(p, m, n, h_tiles, d_packed, stream=None):
    """h_tiles: numpy uint8 (m/16, n/16, 32k) logical tiles; d_packed: torch uint8 CUDA tensor."""
    h = np.ascontiguousarray(h_tiles, dtype=np.uint8)
    assert h.size == (m // 16) * (n // 16) * 32 * p.k
    _check("qtip_pack", load().qtip_pack(ctypes.byref(p), m, n, h.ctypes.data_as(ctypes.c_void_p), _ptr(d_packed),
                                         _stream(stream)))


def qtip_pack_states(p, m, n, h_states, d_packed, stream=None):
    h = np.ascontiguousarray(h_states, dtype=np.uint32)
    _check("qtip_pack_states", load().qtip_pack_states(ctypes.byref(p), m, n, h.ctypes.data_as(ctypes.c_void_p),
                                                       _ptr(d_packed), _stream(stream)))


def qtip_decode(p, m, n, d_packed, d_lut, d_out, out_f32=False, stream=None):
    _check("qtip_decode", load().qtip_decode(ctypes.byref(p), m, n, _ptr(d_packed), _ptr(d_lut), int(out_f32),
                                             _ptr(d_out), _stream(stream)))


def workspace_bytes(p, m, n, B):
    return load().qtip_matvec_workspace_bytes(ctypes.byref(p), m, n, B)


def qtip_matvec(p, m, n, B, d_packed, d_lut, d_sign_n, d_sign_m, scale, d_x, d_y, row_begin=0, row_end=None,
                flags=QTIP_RHT_IN | QTIP_RHT_OUT, d_workspace=None, stream=None):
    row_end = m if row_end is None else row_end
    ws_bytes = d_workspace.numel() * d_workspace.element_size()
    _check("qtip_matvec", load().qtip_matvec(ctypes.byref(p), m, n, B, _ptr(d_packed), _ptr(d_lut), _ptr(d_sign_n),
                                             _ptr(d_sign_m), float(scale), _ptr(d_x), _ptr(d_y), row_begin, row_end,
                                             flags, _ptr(d_workspace), ws_bytes, _stream(stream)))


def qtip_matvec_group(p, m, n, B, d_packed, d_lut, d_sign_n, d_sign_m, scales, d_x, d_y,
                      flags=QTIP_RHT_IN | QTIP_RHT_OUT, d_workspace=None, stream=None):
    """G same-shape layers on one input (lists of device tensors, one entry per layer)."""
    G = len(d_packed)
    arr = lambda ts: (ctypes.c_void_p * G)(*[_ptr(t) for t in ts])
    ws_bytes = min(w.numel() * w.element_size() for w in d_workspace)
    _check("qtip_matvec_group", load().qtip_matvec_group(
        ctypes.byref(p), G, m, n, B, arr(d_packed), None if d_lut is None else arr(d_lut), arr(d_sign_n), arr(d_sign_m),
        (ctypes.c_float * G)(*[float(v) for v in scales]), _ptr(d_x), arr(d_y), flags, arr(d_workspace), ws_bytes,
        _stream(stream)))


def group_fused(p, G, m, n, B):
    """True if qtip_matvec_group runs these G layers as the grouped launches."""
    return bool(load().qtip_matvec_group_fused(ctypes.byref(p), G, m, n, B))


def viterbi_workspace_bytes(p, T):
    return int(load().qtip_viterbi_workspace_bytes(ctypes.byref(p), T))


def qtip_viterbi_tailbite(p, nseq, T, d_source, d_states, d_cost, d_workspace, d_lut=None, stream=None):
    """Algorithm 4 on nseq device sequences (float32 [nseq][T], code units) -> device walks
    (uint32 [nseq][T/V]) and costs (float32 [nseq]); d_lut: HYB binary16 pairs."""
    _check("qtip_viterbi_tailbite", load().qtip_viterbi_tailbite(
        ctypes.byref(p), nseq, T, _ptr(d_source), _ptr(d_lut), _ptr(d_states), _ptr(d_cost), _ptr(d_workspace),
        d_workspace.numel() * d_workspace.element_size(), _stream(stream)))


def quantize_workspace_bytes(p, m, n):
    return int(load().qtip_quantize_workspace_bytes(ctypes.byref(p), m, n))


def qtip_quantize_matrix(p, m, n, d_W, source_scale, d_states, d_cost, d_workspace, d_lut=None, stream=None):
    _check("qtip_quantize_matrix", load().qtip_quantize_matrix(
        ctypes.byref(p), m, n, _ptr(d_W), float(source_scale), _ptr(d_lut), _ptr(d_states), _ptr(d_cost),
        _ptr(d_workspace), d_workspace.numel() * d_workspace.element_size(), _stream(stream)))


def qtip_chain_plan_create(p, layers, B, d_lut=None):
    """layers: list of dicts (packed, sign_n, sign_m: device tensors; scale; m; n; y: device
    float32 (B, m); stage; src) in stage order -> opaque plan handle (c_void_p)."""
    arr = (ChainLayer * len(layers))()
    for i, d in enumerate(layers):
        arr[i] = ChainLayer(d["packed"].data_ptr(), d["sign_n"].data_ptr(), d["sign_m"].data_ptr(), float(d["scale"]),
                            int(d["m"]), int(d["n"]), d["y"].data_ptr(), int(d["stage"]), int(d["src"]))
    plan = ctypes.c_void_p()
    _check("qtip_chain_plan_create", load().qtip_chain_plan_create(ctypes.byref(p), len(layers), arr, int(B),
                                                                   _ptr(d_lut), ctypes.byref(plan)))
    return plan


def qtip_chain_run(plan, d_x, stream=None):
    _check("qtip_chain_run", load().qtip_chain_run(plan, _ptr(d_x), _stream(stream)))


def qtip_chain_plan_destroy(plan):
    if plan:
        load().qtip_chain_plan_destroy(plan)


def qtip_rht(n, B, d_sign, d_in, d_out, inverse=False, stream=None):
    _check("qtip_rht", load().qtip_rht(n, B, _ptr(d_sign), _ptr(d_in), _ptr(d_out), int(inverse), _stream(stream)))


def hadamard_order(n):
    b, a = ctypes.c_int32(), ctypes.c_int32()
    _check("qtip_hadamard_order", load().qtip_hadamard_order(n, ctypes.byref(b), ctypes.byref(a)))
    return b.value, a.value


def set_matvec_impl(impl):
    load().qtip_set_matvec_impl(int(impl))


def get_matvec_impl():
    return load().qtip_get_matvec_impl()


def launch_count():
    return load().qtip_launch_count()


def profile_events(ev_start, ev_stop):
    """Arm the next qtip_matvec on this thread to record torch.cuda.Event pair around its GEMV kernel."""
    if ev_start is None:
        load().qtip_profile_events(None, None)
        return
    for ev in (ev_start, ev_stop):
        if not ev.cuda_event:
            ev.record()                       # torch creates the cudaEvent_t lazily
    load().qtip_profile_events(ctypes.c_void_p(ev_start.cuda_event), ctypes.c_void_p(ev_stop.cuda_event))


def set_pdl(enable):
    load().qtip_set_pdl(int(bool(enable)))


def paley_host(b):
    """The library's own Paley-I matrix (host copy), for orthogonality tests."""
    lib = load()
    fn = lib.qtip_internal_paley_host
    fn.argtypes = [ctypes.c_int, ctypes.c_void_p]
    fn.restype = ctypes.c_int
    out = np.zeros((b, b), dtype=np.int8)
    if fn(b, out.ctypes.data_as(ctypes.c_void_p)) != 0:
        raise ValueError(f"unsupported Paley order {b}")
    return out
