"""QTIPQuantizer: tail-biting trellis quantization of RHT-domain weight tiles on the GPU
(Algorithm 4), producing the packed stream QTIPLinear decodes.

All arithmetic runs in libqtip (qtip_viterbi_tailbite / qtip_quantize_matrix, k_viterbi.cu): the
block scan of P:833 and the scaling into code units (reading R9) happen in the library's gather
kernel; this module only moves buffers and hands the walks to qtip_pack_states.
"""
import numpy as np
import torch

from . import qtip


class QTIPQuantizer:
    def __init__(self, code="3inst", k=2, device="cuda", lut=None):
        """lut: HYB only, numpy uint16 (2^9, 2) binary16 pairs (the table the layer decodes with)."""
        self.code, self.k = code, k
        self.p = qtip.params_default(code, k)
        self.V = 2 if code == "hyb" else 1
        self.device = torch.device(device)
        self.lut = None
        if code == "hyb":
            if lut is None:
                raise ValueError("HYB needs a LUT")
            self.lut = torch.from_numpy(np.ascontiguousarray(lut, dtype=np.uint16).view(np.int16)).to(self.device)
        self._ws = {}

    def workspace(self, T):
        if T not in self._ws:
            self._ws[T] = torch.empty(qtip.viterbi_workspace_bytes(self.p, T), dtype=torch.uint8, device=self.device)
        return self._ws[T]

    def encode(self, src_code_units):
        """src_code_units: float32 CUDA [nseq][T] (already multiplied by the code's state std).
        Returns (walks uint32 CUDA [nseq][T], costs float32 CUDA [nseq])."""
        assert src_code_units.dtype == torch.float32 and src_code_units.is_cuda and src_code_units.is_contiguous()
        nseq, T = src_code_units.shape
        states = torch.empty((nseq, T // self.V), dtype=torch.int32, device=self.device)
        cost = torch.empty(nseq, dtype=torch.float32, device=self.device)
        if nseq == 0:                               # no sequences: nothing to encode, no launch
            return states, cost
        qtip.qtip_viterbi_tailbite(self.p, nseq, T, src_code_units, states, cost, self.workspace(T), d_lut=self.lut)
        return states, cost

    def quantize_tiles(self, W_tilde, code_std):
        """W_tilde: float32 [m][n] RHT-domain weights (m, n multiples of 16), each 16 x 16 tile one
        T = 256 sequence in row-major scan, scaled by code_std into code units in
        the library (qtip_quantize_matrix).  Returns the host walks (uint32 [m/16][n/16][256/V]) for
        qtip_pack_states and the per-tile costs (CUDA)."""
        m, n = W_tilde.shape
        W = W_tilde.to(device=self.device, dtype=torch.float32).contiguous()
        states = torch.empty((m // 16, n // 16, 256 // self.V), dtype=torch.int32, device=self.device)
        cost = torch.empty((m // 16, n // 16), dtype=torch.float32, device=self.device)
        ws = torch.empty(qtip.quantize_workspace_bytes(self.p, m, n), dtype=torch.uint8, device=self.device)
        qtip.qtip_quantize_matrix(self.p, m, n, W, code_std, states, cost, ws, d_lut=self.lut)
        return states.cpu().numpy().astype(np.uint32), cost.reshape(-1)
