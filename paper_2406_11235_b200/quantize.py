"""QTIPQuantizer: tail-biting trellis quantization of RHT-domain weight tiles on the GPU
(Algorithm 4), producing the packed stream QTIPLinear decodes.

All arithmetic runs in libqtip (qtip_viterbi_tailbite / qtip_quantize_matrix, k_viterbi.cu): the
block scan of P:833 and the scaling into code units (reading R9) happen in the library's gather
kernel; this module only moves buffers and hands the walks to qtip_pack_states.

blockldlq() drives Algorithm 5 (BlockLDLQ with QTIP rounding) on the GPU: the one-off
T_y-block LDL factorisation and the per-column error-feedback product are plain library linear
algebra (cuSOLVER Cholesky and a cuBLAS fp32 GEMM through torch), every rounding step is the
library's Algorithm 4 (qtip_quantize_matrix) and every reconstruction its decoder (qtip_pack_states
+ qtip_decode).
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

    def blockldlq(self, W_tilde, H_tilde, code_std, Ty=16):
        """Algorithm 5 with T_x = T_y = 16 (one 16 x 16 tile = one T = 256 sequence, the
        layout QTIPLinear decodes): W~ [m][n] RHT-domain weights, H~ [n][n] the RHT-domain proxy
        Hessian (PSD).  H = L D L^T (T_y-block LDL: L = C blockdiag(C_jj)^-1 from the Cholesky factor
        C, unit lower block-triangular), A = L - I; right to left over block columns j:
            x = W[:, j] + (W[:, jT_y:] - W^[:, jT_y:]) A[jT_y:, j],   W^[:, j] = decode(Viterbi(x)) / code_std.
        Returns (W^ float32 CUDA [m][n], walks uint32 [n/T_y][m/16][256/V] host)."""
        if Ty != 16:
            raise ValueError("blockldlq: T_y = 16 (the 16 x 16 tile of the packed layout)")
        if torch.backends.cuda.matmul.allow_tf32:
            raise RuntimeError("blockldlq: TF32 matmul is enabled; the feedback product needs fp32")
        dev = self.device
        W = W_tilde.to(device=dev, dtype=torch.float32).contiguous()
        m, n = W.shape
        H = torch.as_tensor(H_tilde, dtype=torch.float64, device=dev)
        nb = n // Ty
        C = torch.linalg.cholesky(H)                                         # H = C C^T
        Cd = torch.stack([C[j * Ty:(j + 1) * Ty, j * Ty:(j + 1) * Ty] for j in range(nb)])
        Cdi = torch.linalg.inv(Cd)
        Lm = torch.cat([C[:, j * Ty:(j + 1) * Ty] @ Cdi[j] for j in range(nb)], dim=1)
        A = (Lm - torch.eye(n, dtype=torch.float64, device=dev)).to(torch.float32)
        What = torch.zeros((m, n), dtype=torch.float32, device=dev)
        states = torch.empty((m // 16, 1, 256 // self.V), dtype=torch.int32, device=dev)
        cost = torch.empty((m // 16, 1), dtype=torch.float32, device=dev)
        ws = torch.empty(qtip.quantize_workspace_bytes(self.p, m, Ty), dtype=torch.uint8, device=dev)
        packed = torch.empty(qtip.packed_bytes(self.p, m, Ty), dtype=torch.uint8, device=dev)
        dec = torch.empty((m, Ty), dtype=torch.float16, device=dev)
        walks = np.empty((nb, m // 16, 256 // self.V), dtype=np.uint32)
        for j in range(nb - 1, -1, -1):
            c0, c1 = j * Ty, (j + 1) * Ty
            x = (W[:, c0:c1] + (W[:, c0:] - What[:, c0:]) @ A[c0:, c0:c1]).contiguous()
            qtip.qtip_quantize_matrix(self.p, m, Ty, x, code_std, states, cost, ws, d_lut=self.lut)
            h = states.cpu().numpy().astype(np.uint32)
            qtip.qtip_pack_states(self.p, m, Ty, h, packed)
            qtip.qtip_decode(self.p, m, Ty, packed, self.lut, dec)
            What[:, c0:c1] = dec.float() / code_std
            walks[j] = h.reshape(m // 16, -1)
        return What, walks
