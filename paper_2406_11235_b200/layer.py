"""QTIPLinear: one QTIP-quantized linear layer y = W x on the GPU (the call a user makes).

W = scale * S_m H_m^T W~ H_n S_n with W~ stored as packed trellis tiles.
Holds device buffers (packed stream, signs, LUT, workspace) and calls qtip_matvec; all
arithmetic happens in libqtip.
"""
import numpy as np
import torch

from . import qtip


class QTIPLinear:
    def __init__(self, m, n, code="3inst", k=2, device="cuda", two_sign=False):
        self.m, self.n, self.code, self.k = m, n, code, k
        self.device = torch.device(device)
        self.p = qtip.params_default(code, k, two_sign)
        nbytes = qtip.packed_bytes(self.p, m, n)
        if nbytes < 0:
            raise ValueError(f"unsupported QTIP config {code} k={k} for {m}x{n}")
        self.packed = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)
        self.sign_m = torch.zeros((m + 7) // 8, dtype=torch.uint8, device=self.device)
        self.sign_n = torch.zeros((n + 7) // 8, dtype=torch.uint8, device=self.device)
        self.lut = None
        self.scale = 1.0
        self._ws = {}

    # ------------------------------------------------------------------ loading
    def load_tiles(self, tiles, sign_m, sign_n, scale=1.0, lut=None):
        """tiles: numpy uint8 (m/Tx, n/Ty, 32k) logical tail-biting streams; signs: bit-packed
        numpy uint8; lut: numpy uint16 binary16 -- (2^Q, 2) for HYB, (2^Q,) for "hyb1", (2^L,) for "lut"."""
        qtip.qtip_pack(self.p, self.m, self.n, tiles, self.packed)
        self.sign_m.copy_(torch.from_numpy(np.ascontiguousarray(sign_m, dtype=np.uint8)))
        self.sign_n.copy_(torch.from_numpy(np.ascontiguousarray(sign_n, dtype=np.uint8)))
        if self.code in ("hyb", "hyb1", "lut"):
            if lut is None:
                raise ValueError(f"{self.code} needs a LUT")
            self.lut = torch.from_numpy(np.ascontiguousarray(lut, dtype=np.uint16).view(np.int16)).to(self.device)
        self.scale = float(scale)
        return self

    def workspace(self, B):
        if B not in self._ws:
            nb = qtip.workspace_bytes(self.p, self.m, self.n, B)
            self._ws[B] = torch.zeros(nb, dtype=torch.uint8, device=self.device)   # grid-barrier counters start at 0
        return self._ws[B]

    # ------------------------------------------------------------------ compute
    def forward(self, x, out=None, flags=qtip.QTIP_RHT_IN | qtip.QTIP_RHT_OUT, rows=None, stream=None):
        """x: float32 CUDA (B, n) -> float32 (B, m) (or the row range of scale * W~ x~)."""
        _check_io(x, (x.shape[0] if x.dim() == 2 else -1, self.n), self.device, "x")
        B = x.shape[0]
        r0, r1 = rows if rows is not None else (0, self.m)
        if out is None:
            out = torch.empty((B, r1 - r0), dtype=torch.float32, device=self.device)
        _check_io(out, (B, r1 - r0), self.device, "out")
        if B == 0:                                  # empty batch: nothing to compute, no launch
            return out
        qtip.qtip_matvec(self.p, self.m, self.n, B, self.packed, self.lut, self.sign_n, self.sign_m, self.scale,
                         x, out, r0, r1, flags, self.workspace(B), stream)
        return out

    __call__ = forward

    def decode(self, out_f32=False):
        out = torch.empty((self.m, self.n), dtype=torch.float32 if out_f32 else torch.float16, device=self.device)
        qtip.qtip_decode(self.p, self.m, self.n, self.packed, self.lut, out, out_f32)
        return out

    @property
    def stream_bytes(self):
        """Algorithmic compressed bytes m n k / 8 (the metric's numerator)."""
        return self.m * self.n * self.k // 8


def _check_io(t, shape, device, name):
    """The C ABI receives raw pointers: shapes, dtype, layout and device are checked here."""
    if not (isinstance(t, torch.Tensor) and t.dtype == torch.float32 and t.is_cuda and t.is_contiguous()):
        raise ValueError(f"{name}: a contiguous float32 CUDA tensor is required")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")
    if t.device != device and not (device.index is None and t.device.type == device.type):
        raise ValueError(f"{name}: on {t.device}, the layer is on {device}")


_SIDE = {}


def _side_streams(device, count):
    lst = _SIDE.setdefault(str(device), [])
    while len(lst) < count:
        lst.append(torch.cuda.Stream(device=device))
    return lst[:count]


def forward_group(layers, x, outs=None, flags=qtip.QTIP_RHT_IN | qtip.QTIP_RHT_OUT, stream=None):
    """Same-shape QTIPLinear layers applied to one input x (e.g. q, k, v): one qtip_matvec_group
    call (grouped RHT-in, one persistent decode-GEMV launch over all layers, grouped RHT-out)."""
    l0 = layers[0]
    for l in layers[1:]:
        if (l.m, l.n, l.code, l.k) != (l0.m, l0.n, l0.code, l0.k) or bytes(l.p) != bytes(l0.p):
            raise ValueError("forward_group: layers must share shape and QTIP parameters")
    _check_io(x, (x.shape[0] if x.dim() == 2 else -1, l0.n), l0.device, "x")
    B = x.shape[0]
    if outs is None:
        outs = [torch.empty((B, l.m), dtype=torch.float32, device=l.device) for l in layers]
    if len(outs) != len(layers):
        raise ValueError("forward_group: one output per layer")
    for l, o in zip(layers, outs):
        _check_io(o, (B, l.m), l.device, "outs[]")
    if B == 0:                                      # empty batch: nothing to compute, no launch
        return outs
    if len(layers) > 1 and stream is None and not qtip.group_fused(l0.p, len(layers), l0.m, l0.n, B):
        # no grouped launch for this shape / batch: the layers run concurrently on side streams
        cur = torch.cuda.current_stream(l0.device)
        side = _side_streams(l0.device, len(layers) - 1)
        for s in side:
            s.wait_stream(cur)
        layers[0].forward(x, out=outs[0], flags=flags)
        for s, l, o in zip(side, layers[1:], outs[1:]):
            with torch.cuda.stream(s):
                l.forward(x, out=o, flags=flags)
        for s in side:
            cur.wait_stream(s)
        return outs
    qtip.qtip_matvec_group(l0.p, l0.m, l0.n, B, [l.packed for l in layers],
                           [l.lut for l in layers] if l0.code == "hyb" else None,
                           [l.sign_n for l in layers], [l.sign_m for l in layers], [l.scale for l in layers], x, outs,
                           flags, [l.workspace(B) for l in layers], stream)
    return outs



class QTIPChain:
    """A chain of QTIPLinear layers run as ONE persistent launch per call (qtip_chain_run): stage 0
    reads the external x, every later stage reads the output of one layer of the previous stage
    (e.g. a decode step: q, k, v -> o -> gate, up -> down -> ...).

    stages: list of (layers, src) with layers a list of QTIPLinear sharing n, and src the index
    (within the previous stage) of the layer whose output is this stage's input (ignored for
    stage 0).  Outputs: self.outs[stage][i], float32 (B, m), rewritten by every call."""

    def __init__(self, stages, B=1):
        if not stages:
            raise ValueError("QTIPChain: no stages")
        l0 = stages[0][0][0]
        self.B, self.device, self.p = B, l0.device, l0.p
        self.outs, descs, first = [], [], []
        for si, (layers, src) in enumerate(stages):
            outs = []
            if si > 0 and not 0 <= int(src) < len(stages[si - 1][0]):
                raise ValueError(f"QTIPChain: stage {si} src {src} is not a layer of stage {si - 1}")
            first.append(len(descs))
            for lay in layers:
                if bytes(lay.p) != bytes(l0.p):
                    raise ValueError("QTIPChain: all layers share the QTIP parameters")
                y = torch.empty((B, lay.m), dtype=torch.float32, device=self.device)
                outs.append(y)
                descs.append(dict(packed=lay.packed, sign_n=lay.sign_n, sign_m=lay.sign_m, scale=lay.scale, m=lay.m,
                                  n=lay.n, y=y, stage=si, src=-1 if si == 0 else first[si - 1] + int(src)))
            self.outs.append(outs)
        self.n_in = stages[0][0][0].n
        self.layers = [lay for layers, _ in stages for lay in layers]
        lut = l0.lut if l0.code == "hyb" else None
        self._plan = qtip.qtip_chain_plan_create(self.p, descs, B, lut)

    def forward(self, x, stream=None):
        _check_io(x, (self.B, self.n_in), self.device, "x")
        qtip.qtip_chain_run(self._plan, x, stream)
        return self.outs

    __call__ = forward

    def close(self):
        if getattr(self, "_plan", None):
            qtip.qtip_chain_plan_destroy(self._plan)
            self._plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:       # noqa: BLE001  (interpreter shutdown)
            pass
