"""Dense decode of a QTIP-packed matrix and the float64 matrix-vector product.  (oracle; test infrastructure only)

Paper passages:
  P:389-390  a T_x x T_y block of weights is quantized as one sequence; T_x = T_y = 16.
  P:833      x.reshape(m/T_x, T_x T_y): the sequence of a block is its rows concatenated
             (row-major scan, reading R5): position p = 16 r + c.
  P:121-123  the reconstruction concatenates node values along the walk (V values per node).
  P:96-97    RHT: W = S_m H_m^T W~ H_n S_n (orthonormal H), see oracle.rht.

  P:787-791  the lookup-only code uses T_x = 32, T_y = 8 blocks: position p = 8 r + c.

The plain definition this module writes out:
    W~[T_x I + r, T_y J + c] = code(state_p(tile I,J)),  p = T_y r + c   (V = 1)
    (W~[.., 2t], W~[.., 2t+1]) = code(state_t)                       (V = 2, HYB)
    y = scale * S_m H_m^T W~ H_n S_n x   evaluated in float64.
Logical tile format: kT bits, MSB-first (oracle.trellis), i.e. 32k bytes per tile,
tiles indexed [I, J] (tile-row major).
"""
from dataclasses import dataclass
import numpy as np

from . import codes, rht, trellis

TX = TY = 16
T = TX * TY


@dataclass
class Params:
    L: int = 16
    k: int = 2
    V: int = 1
    code: str = "3inst"          # "1mad" | "3inst" | "hyb" (V = 2) | "hyb1" (HYB, V = 1) | "lut"
    Q: int = 9
    lut: np.ndarray = None       # uint16 (2^Q, 2) for HYB, (2^Q,) for hyb1, (2^L,) for lut
    two_sign: bool = False
    tail_biting: bool = True
    Tx: int = 16
    Ty: int = 16


def tile_values(tile_bytes, p: Params):
    """float64 (..., 256) values of tiles (..., 32k bytes), in sequence order p = 16 r + c."""
    st = trellis.tile_states(tile_bytes, p.L, p.k, p.V, T)          # (..., T/V)
    if p.code == "1mad":
        v = codes.f16_to_f64(codes.decode_1mad(st.astype(np.uint64)))
    elif p.code == "3inst":
        v = codes.f16_to_f64(codes.decode_3inst(st.astype(np.uint64)))
    elif p.code == "hyb":
        v = codes.f16_to_f64(codes.decode_hyb(st.astype(np.uint64), p.lut, p.Q, p.two_sign))
        v = v.reshape(v.shape[:-2] + (T,))                         # (t, 2) -> positions 2t, 2t+1
    elif p.code == "hyb1":
        v = codes.f16_to_f64(codes.decode_hyb1(st.astype(np.uint64), p.lut, p.Q))
    elif p.code == "lut":
        v = codes.f16_to_f64(codes.decode_lut(st, p.lut))
    else:
        raise ValueError(p.code)
    return v


def dense_decode(tiles, p: Params):
    """tiles: uint8 (m/Tx, n/Ty, 32k) -> float64 W~ (m, n) (exact fp16 values)."""
    tiles = np.asarray(tiles, dtype=np.uint8)
    mt, nt = tiles.shape[:2]
    v = tile_values(tiles, p).reshape(mt, nt, p.Tx, p.Ty)           # [I, J, r, c]
    return v.transpose(0, 2, 1, 3).reshape(mt * p.Tx, nt * p.Ty)


def decode_rows(tiles, p: Params, rows):
    """Only the listed rows of W~ (for full-size sampled parity checks)."""
    tiles = np.asarray(tiles, dtype=np.uint8)
    out = []
    for i in rows:
        I, r = divmod(int(i), p.Tx)
        v = tile_values(tiles[I], p).reshape(-1, p.Tx, p.Ty)        # [J, r, c]
        out.append(v[:, r, :].reshape(-1))
    return np.stack(out)


def matvec(Wt, x, sign_n=None, sign_m=None, scale=1.0, rht_in=True, rht_out=True, rows=None):
    """y[b] = scale * S_m H_m^T W~ H_n S_n x[b]  (float64).

    Wt: decoded W~ (m, n) float64; x: (B, n).  Without rht_in x~ = x; without rht_out the
    result is scale * W~ x~.  rows=(r0, r1) selects output rows (requires rht_out=False,
    since H_m^T mixes all rows)."""
    if rows is not None and rht_out:
        raise ValueError("a row range needs rht_out=False")
    Wt = np.asarray(Wt, dtype=np.float64)
    m, n = Wt.shape
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    xt = rht.rht_forward(x, sign_n, n) if rht_in else x
    yt = xt @ Wt.T                                                   # (B, m)
    if rows is not None:
        return scale * yt[:, rows[0]:rows[1]]
    if rht_out:
        yt = rht.rht_inverse(yt, sign_m, m)
    return scale * yt


def xtilde(x, sign_n, n):
    return rht.rht_forward(np.atleast_2d(x), sign_n, n)
