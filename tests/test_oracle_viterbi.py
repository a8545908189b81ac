"""Pins for oracle.viterbi: Fig. 2, brute force on tiny trellises, constraint
dominance, Alg. 4 >= the exact tail-biting optimum, and the paper's Tables 1 and 3."""
import json
import os

import numpy as np
import pytest

from oracle import codes, trellis, viterbi

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_fig2_viterbi_exact():
    g = _load("fig2.json")
    st, cost = viterbi.viterbi(g["reconstruction"], g["L"], g["k"], g["V"], np.array(g["node_values"]))
    assert cost == 0.0
    assert list(st) == g["walk"]


def test_constant_code_ties_to_smallest_states():
    s = np.array([0.3, -1.0, 2.0, 0.5])
    st, cost = viterbi.viterbi(s, 4, 1, 1, np.full(16, 0.25))
    assert list(st) == [0, 0, 0, 0]
    assert np.isclose(cost, ((s - 0.25) ** 2).sum())


@pytest.mark.parametrize("L,k,V,T", [(4, 1, 1, 8), (5, 2, 1, 6), (6, 2, 2, 6), (4, 2, 2, 6), (3, 1, 1, 7)])
def test_dp_equals_brute_force(L, k, V, T):
    rng = np.random.default_rng(L * 100 + k * 10 + T)
    for trial in range(4):
        tab = rng.standard_normal((1 << L) * V)
        s = rng.standard_normal(T)
        st, c = viterbi.viterbi(s, L, k, V, tab)
        bst, bc = viterbi.brute_force(s, L, k, V, tab)
        assert c == bc                                  # exact: same left-to-right float64 sums
        assert list(st) == list(bst)
        assert trellis.is_walk(list(st), L, k, V)


def test_dp_tie_rule_on_forced_ties():
    """Integer code + integer source force many exact ties; the DP's smallest-index rule must pick
    the reverse-lexicographic minimum among optimal walks (reading R4)."""
    rng = np.random.default_rng(11)
    L, k, V, T = 4, 1, 1, 7
    for trial in range(40):
        tab = rng.integers(-2, 3, 1 << L).astype(np.float64)
        s = rng.integers(-2, 3, T).astype(np.float64)
        st, c = viterbi.viterbi(s, L, k, V, tab)
        bst, bc = viterbi.brute_force(s, L, k, V, tab)
        assert c == bc and list(st) == list(bst)


def test_constrained_dominance_and_exact_tailbite_equals_brute_force():
    rng = np.random.default_rng(12)
    L, k, V, T = 4, 1, 1, 8
    for trial in range(4):
        tab = rng.standard_normal(1 << L)
        s = rng.standard_normal(T)
        _, free = viterbi.viterbi(s, L, k, V, tab)
        costs = []
        for O in range(1 << (L - k * V)):
            st, c = viterbi.viterbi(s, L, k, V, tab, overlap=O)
            assert c >= free
            assert trellis.is_walk(list(st), L, k, V, tail_biting=True)
            assert (int(st[0]) >> (k * V)) == O and (int(st[-1]) & ((1 << (L - k * V)) - 1)) == O
            costs.append(c)
        est, ec = viterbi.exact_tailbite(s, L, k, V, tab)
        bst, bc = viterbi.brute_force(s, L, k, V, tab, tail_biting=True)
        assert np.isclose(ec, bc, rtol=0, atol=1e-12) and ec == min(costs)


def test_constraint_inactive_at_own_overlap():
    rng = np.random.default_rng(13)
    L, k, V = 6, 2, 1
    tab = rng.standard_normal(1 << L)
    s = rng.standard_normal(10)
    st, c = viterbi.viterbi(s, L, k, V, tab)
    if (int(st[0]) >> (k * V)) == (int(st[-1]) & ((1 << (L - k * V)) - 1)):
        st2, c2 = viterbi.viterbi(s, L, k, V, tab, overlap=int(st[0]) >> (k * V))
        assert c2 == c and list(st2) == list(st)


def test_alg4_is_tail_biting_and_no_better_than_exact():
    rng = np.random.default_rng(14)
    for (L, k, V, T) in [(6, 1, 1, 16), (6, 2, 1, 16), (8, 2, 2, 16)]:
        tab = rng.standard_normal((1 << L) * V)
        for trial in range(5):
            s = rng.standard_normal(T)
            st, c = viterbi.tailbite_encode(s, L, k, V, tab)
            assert trellis.is_walk(list(st), L, k, V, tail_biting=True)
            _, ec = viterbi.exact_tailbite(s, L, k, V, tab)
            assert c >= ec - 1e-12
            # the walk packs to exactly kT bits and unpacks back
            bits = trellis.pack([int(v) for v in st], L, k, V, tail_biting=True)
            assert len(bits) == k * T
            assert trellis.unpack(bits, L, k, V, T // V, tail_biting=True) == [int(v) for v in st]
            assert np.isclose(((viterbi.reconstruct(st, tab, L, V) - s) ** 2).sum(), c)


def test_alg4_seam_reading():
    """Alg. 4 line 3 reads the overlap between rotated groups floor(T/(2V)) and +1 (1-indexed)."""
    st = np.array([0b101100, 0b110011, 0b001110, 0b111000], dtype=np.uint32)   # L=6, kV=2, 4 groups
    assert viterbi.seam_overlap(st, 8, 6, 1, 2) == 0b110011 & 0b1111            # T=8, V=2 -> group 2


@pytest.mark.slow
def test_table3_alg4_reproduction():
    """P:356-370 Table 3: Alg. 4 MSE with a tail-biting (12, k, 1) trellis, T = 256, i.i.d. N(0,1),
    random N(0,1) lookup code (the paper does not fix the code; any Gaussian LUT)."""
    ref = _load("paper_tables.json")["table3"]
    rng = np.random.default_rng(5000)
    lut = rng.standard_normal(1 << 12)
    nseq = 384
    for k in (1, 2, 3, 4):
        S = rng.standard_normal((nseq, 256))
        st, c = viterbi.tailbite_encode_batch(S, 12, k, 1, lut)
        mse = c / 256
        se = mse.std() / np.sqrt(nseq)
        paper = ref["alg4_mse"][str(k)]
        assert abs(mse.mean() - paper) <= 3 * se + 0.0006, (k, mse.mean(), paper, se)
        assert mse.mean() > codes.distortion_rate_bound(k)


@pytest.mark.slow
def test_table1_computed_codes_reproduction():
    """P:224-235 Table 1 (k=2, L=16, T=256): 1MAD 0.069, 3INST 0.069, HYB 0.071, all above D_R = 0.0625.
    Reading R9: the quantizer uses the code divided by its std over all 2^L states (the scale is
    folded into the per-matrix scale); Table 1 is read as tail-biting (Alg. 4)."""
    ref = _load("paper_tables.json")["table1"]["mse"]
    nseq = 64
    S = np.random.default_rng(5000).standard_normal((nseq, 256))
    lut = codes.kmeans_lut(9, seed=4000, n_samples=1 << 16, iters=15)
    for name, V in (("1mad", 1), ("3inst", 1), ("hyb", 2)):
        tab = codes.code_table(name, 16, lut=lut, Q=9)
        tab = tab / tab.std()
        st, c = viterbi.tailbite_encode_batch(S, 16, 2, V, tab)
        mse = c / 256
        se = mse.std() / np.sqrt(nseq)
        assert abs(mse.mean() - ref[name]) <= 3 * se + 0.0015, (name, mse.mean(), ref[name], se)
        assert mse.mean() > ref["d_r"]
