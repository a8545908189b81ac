"""Trellis quantizer: Viterbi, Alg. 4 tail-biting approximation,
brute force and the exact tail-biting optimum.  (oracle; test infrastructure only)

The DP itself is plain C (viterbi.c, built with gcc on first use or by
__graft_entry__.build()); Alg. 4 is written here step by step in the paper's order.
"""
import ctypes
import itertools
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "viterbi.c")
_LIB = os.path.join(_HERE, "_viterbi.so")
_lib = None


def build(force=False):
    """Compile viterbi.c -> _viterbi.so (plain gcc; OpenMP over independent sequences)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        _lib.qo_viterbi.restype = ctypes.c_double
        _lib.qo_viterbi.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long,
                                                          ctypes.c_void_p]
        _lib.qo_viterbi_batch.restype = None
        _lib.qo_viterbi_batch.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p, ctypes.c_int] + [ctypes.c_void_p] * 4
        _lib.qo_viterbi_f32.restype = ctypes.c_float
        _lib.qo_viterbi_f32.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long,
                                                              ctypes.c_void_p]
        _lib.qo_viterbi_f32_batch.restype = None
        _lib.qo_viterbi_f32_batch.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p, ctypes.c_int] + [ctypes.c_void_p] * 4
    return _lib


def _table(code_table, L, V):
    t = np.ascontiguousarray(np.asarray(code_table, dtype=np.float64).reshape(1 << L, V))
    return t


def viterbi(s, L, k, V, code_table, overlap=None):
    """Optimal walk for source s (length T, T % V == 0); overlap = tail-biting constraint O or None.
    Returns (states uint32 (T/V,), cost float)."""
    lib = _load()
    s = np.ascontiguousarray(np.asarray(s, dtype=np.float64))
    if len(s) % V:
        raise ValueError("T must be divisible by V")
    n = len(s) // V
    tab = _table(code_table, L, V)
    out = np.zeros(n, dtype=np.uint32)
    cost = lib.qo_viterbi(L, k * V, V, n, tab.ctypes.data, s.ctypes.data, -1 if overlap is None else int(overlap),
                          out.ctypes.data)
    if cost < 0:
        raise MemoryError
    return out, cost


def viterbi_batch(S, L, k, V, code_table, overlaps=None):
    lib = _load()
    S = np.ascontiguousarray(np.asarray(S, dtype=np.float64))
    nseq, T = S.shape
    n = T // V
    tab = _table(code_table, L, V)
    ov = np.full(nseq, -1, dtype=np.int64) if overlaps is None else np.ascontiguousarray(overlaps, dtype=np.int64)
    out = np.zeros((nseq, n), dtype=np.uint32)
    cost = np.zeros(nseq)
    lib.qo_viterbi_batch(L, k * V, V, n, tab.ctypes.data, nseq, S.ctypes.data, ov.ctypes.data, out.ctypes.data,
                         cost.ctypes.data)
    return out, cost


def seam_overlap(states_rot, T, L, k, V):
    """Alg. 4 line 3: the L-kV bit overlap of S'_{floor(T/2)} S'_{floor(T/2)+1} (reading R3:
    1-indexed group floor(T/(2V)); its bottom L-kV bits)."""
    g = T // (2 * V)
    return int(states_rot[g - 1]) & ((1 << (L - k * V)) - 1)


def tailbite_encode(s, L, k, V, code_table):
    """Algorithm 4, in the paper's order."""
    s = np.asarray(s, dtype=np.float64)
    T = len(s)
    s_rot = np.roll(s, T // 2)                                  # rotate S right by floor(T/2)
    states_rot, _ = viterbi(s_rot, L, k, V, code_table)         # S^' <- Viterbi(S', G)
    O = seam_overlap(states_rot, T, L, k, V)                    # overlap at the seam
    return viterbi(s, L, k, V, code_table, overlap=O)           # Viterbi(S, G) with overlap O


def tailbite_encode_batch(S, L, k, V, code_table):
    """Alg. 4 on many independent sequences (same steps, batched DP calls)."""
    S = np.asarray(S, dtype=np.float64)
    T = S.shape[1]
    S_rot = np.roll(S, T // 2, axis=1)
    st_rot, _ = viterbi_batch(S_rot, L, k, V, code_table)
    O = np.array([seam_overlap(r, T, L, k, V) for r in st_rot], dtype=np.int64)
    return viterbi_batch(S, L, k, V, code_table, overlaps=O)


def exact_tailbite(s, L, k, V, code_table):
    """Exact tail-biting optimum: best constrained walk over every overlap O."""
    best = None
    for O in range(1 << (L - k * V)):
        st, c = viterbi(s, L, k, V, code_table, overlap=O)
        if best is None or c < best[1]:
            best = (st, c)
    return best


def brute_force(s, L, k, V, code_table, tail_biting=False):
    """Exhaustive search over all stored bit strings, left-to-right float64 cost,
    ties -> reverse-lexicographic minimum of the walk (the DP's rule, reading R4)."""
    s = np.asarray(s, dtype=np.float64)
    tab = _table(code_table, L, V)
    n = len(s) // V
    kv = k * V
    nbits = kv * n if tail_biting else L + kv * (n - 1)
    best = None
    for bits in itertools.product((0, 1), repeat=nbits):
        states = []
        for t in range(n):
            v = 0
            for i in range(L):
                pos = t * kv + i
                if tail_biting:
                    pos %= nbits
                v = (v << 1) | bits[pos]
            states.append(v)
        cost = 0.0
        for t, y in enumerate(states):
            d = 0.0
            for v in range(V):
                e = tab[y, v] - s[t * V + v]
                d += e * e
            cost += d
        key = (cost, tuple(reversed(states)))
        if best is None or key < best[0]:
            best = (key, states)
    return np.array(best[1], dtype=np.uint32), best[0][0]


def reconstruct(states, code_table, L, V):
    tab = _table(code_table, L, V)
    return tab[np.asarray(states, dtype=np.int64)].reshape(-1)


# ------------------------------------------------------------------ binary32 variant (reading R17)
def viterbi_f32(s, L, k, V, code_table, overlap=None):
    """Viterbi with every cost operation in binary32 (same order as viterbi())."""
    lib = _load()
    s = np.ascontiguousarray(np.asarray(s, dtype=np.float32))
    n = len(s) // V
    tab = np.ascontiguousarray(np.asarray(code_table, dtype=np.float32).reshape(1 << L, V))
    out = np.zeros(n, dtype=np.uint32)
    cost = lib.qo_viterbi_f32(L, k * V, V, n, tab.ctypes.data, s.ctypes.data, -1 if overlap is None else int(overlap),
                              out.ctypes.data)
    return out, float(cost)


def viterbi_f32_batch(S, L, k, V, code_table, overlaps=None):
    lib = _load()
    S = np.ascontiguousarray(np.asarray(S, dtype=np.float32))
    nseq, T = S.shape
    n = T // V
    tab = np.ascontiguousarray(np.asarray(code_table, dtype=np.float32).reshape(1 << L, V))
    ov = np.full(nseq, -1, dtype=np.int64) if overlaps is None else np.ascontiguousarray(overlaps, dtype=np.int64)
    out = np.zeros((nseq, n), dtype=np.uint32)
    cost = np.zeros(nseq, dtype=np.float32)
    lib.qo_viterbi_f32_batch(L, k * V, V, n, tab.ctypes.data, nseq, S.ctypes.data, ov.ctypes.data, out.ctypes.data,
                             cost.ctypes.data)
    return out, cost


def tailbite_encode_f32_batch(S, L, k, V, code_table):
    """Algorithm 4 with the binary32 DP: rotate right by floor(T/2), unconstrained
    Viterbi, seam overlap (reading R3), constrained Viterbi on the original sequence."""
    S = np.asarray(S, dtype=np.float32)
    T = S.shape[1]
    S_rot = np.roll(S, T // 2, axis=1)
    st_rot, _ = viterbi_f32_batch(S_rot, L, k, V, code_table)
    O = np.array([seam_overlap(r, T, L, k, V) for r in st_rot], dtype=np.int64)
    return viterbi_f32_batch(S, L, k, V, code_table, overlaps=O)
