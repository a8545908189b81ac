"""Pins for oracle.trellis: the paper's Fig. 2 worked example, the edge rule and window invariants."""
import json
import os

import numpy as np
import pytest

from oracle import trellis

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def fig2():
    with open(os.path.join(GOLD, "fig2.json")) as f:
        return json.load(f)


def test_next_states_edge_rule():
    # SPEC S:46-48 examples of the P:208 edge rule (L=2, k=1, V=1)
    assert trellis.next_states(0, 2, 1, 1) == [0, 1]
    assert trellis.next_states(1, 2, 1, 1) == [2, 3]
    assert trellis.next_states(3, 2, 1, 1) == [2, 3]
    # every successor shares its top L-kV bits with the bottom L-kV bits of the source
    for L, k, V in [(4, 1, 1), (6, 2, 1), (8, 2, 2), (16, 2, 1)]:
        for i in [0, 1, 5, (1 << L) - 1]:
            nx = trellis.next_states(i, L, k, V)
            assert len(nx) == 1 << (k * V)
            assert all(trellis.is_edge(i, j, L, k, V) for j in nx)
            assert all((j >> (k * V)) == (i & ((1 << (L - k * V)) - 1)) for j in nx)


def test_fig2_pack_unpack():
    g = fig2()
    L, k, V = g["L"], g["k"], g["V"]
    bits = trellis.pack(g["walk"], L, k, V, tail_biting=False)
    assert "".join(map(str, bits)) == g["stored"]
    tb = trellis.pack(g["walk"], L, k, V, tail_biting=True)
    assert "".join(map(str, tb)) == g["stored_tail_biting"]
    stored = np.array([int(c) for c in g["stored"]], dtype=np.uint8)
    assert trellis.unpack(stored, L, k, V, 6, tail_biting=False) == g["walk"]
    stored_tb = np.array([int(c) for c in g["stored_tail_biting"]], dtype=np.uint8)
    assert trellis.unpack(stored_tb, L, k, V, 6, tail_biting=True) == g["walk"]
    vals = [g["node_values"][s] for s in g["walk"]]
    assert vals == g["reconstruction"]


def test_pack_rejects_non_walks():
    with pytest.raises(ValueError):
        trellis.pack([0, 3], 2, 1, 1, tail_biting=False)       # 0 -> 3 is not an edge
    with pytest.raises(ValueError):
        trellis.pack([0, 1], 2, 1, 1, tail_biting=True)        # 1 -> 0 closure fails (1 -> {2,3})


@pytest.mark.parametrize("L,k,V,T", [(16, 2, 1, 256), (16, 4, 2, 256), (16, 3, 2, 256), (16, 3, 1, 256),
                                      (12, 1, 1, 32), (6, 2, 1, 8)])
def test_window_overlap_invariant_with_wrap(L, k, V, T):
    """consecutive windows overlap in L-kV bits; tail-biting wraps."""
    rng = np.random.default_rng(7)
    nb = k * T
    bits = rng.integers(0, 2, size=nb).astype(np.uint8)
    n = T // V
    st = trellis.unpack(bits, L, k, V, n, tail_biting=True)
    assert trellis.is_walk(st, L, k, V, tail_biting=True)
    # window t equals bits [t kV, t kV + L) mod kT read MSB-first
    for t in [0, 1, n // 2, n - 1]:
        ref = 0
        for i in range(L):
            ref = ref * 2 + int(bits[(t * k * V + i) % nb])
        assert st[t] == ref


def test_tile_states_vectorised_matches_windows():
    rng = np.random.default_rng(8)
    for (k, V) in [(2, 1), (4, 2), (3, 2), (3, 1)]:
        tiles = rng.integers(0, 256, size=(3, 32 * k), dtype=np.uint8)
        st = trellis.tile_states(tiles, 16, k, V, 256)
        for i in range(3):
            bits = trellis.bits_from_bytes(tiles[i], 256 * k)
            assert list(st[i]) == trellis.unpack(bits, 16, k, V, 256 // V, tail_biting=True)


def test_pack_unpack_roundtrip_random_walks():
    rng = np.random.default_rng(9)
    for (L, k, V) in [(8, 2, 1), (10, 2, 2), (16, 2, 1), (5, 1, 1)]:
        kv = k * V
        n = 12
        for tb in (False, True):
            bits = rng.integers(0, 2, size=(kv * n if tb else L + kv * (n - 1))).astype(np.uint8)
            walk = trellis.unpack(bits, L, k, V, n, tail_biting=tb)
            assert trellis.is_walk(walk, L, k, V, tail_biting=tb)
            back = trellis.pack(walk, L, k, V, tail_biting=tb)
            assert np.array_equal(back, bits)


def test_tail_biting_strings_biject_onto_closed_walks():
    """Every kT-bit string is a tail-biting walk and vice versa (so random bytes are valid
    packed weights): count closed walks of length n = trace(A^n) = 2^{kVn} (L <= kVn)."""
    L, k, V, n = 3, 1, 1, 5
    N = 1 << L
    A = np.zeros((N, N), dtype=np.int64)
    for i in range(N):
        for j in trellis.next_states(i, L, k, V):
            A[i, j] = 1
    closed = int(np.trace(np.linalg.matrix_power(A, n)))
    assert closed == 2 ** (k * V * n)
    seen = set()
    for v in range(2 ** (k * V * n)):
        bits = np.array(trellis.int_to_bits(v, k * V * n), dtype=np.uint8)
        w = tuple(trellis.unpack(bits, L, k, V, n, tail_biting=True))
        assert trellis.is_walk(list(w), L, k, V, tail_biting=True)
        seen.add(w)
    assert len(seen) == closed
