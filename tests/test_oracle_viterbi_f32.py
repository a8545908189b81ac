"""Pins of the oracle's binary32 Viterbi (oracle/viterbi.c qo_viterbi_f32, reading R17), the
precision the GPU quantizer takes its argmin decisions in.  Pinned against the float64 DP (itself
pinned to brute force in test_oracle_viterbi.py) and against brute force on tiny trellises."""
import numpy as np

from oracle import codes, trellis, viterbi


def _cost64(states, s, tab):
    return float(((tab[np.asarray(states, dtype=np.int64)] - s) ** 2).sum())


def test_f32_matches_brute_force_on_tiny_trellises():
    rng = np.random.default_rng(11)
    for trial in range(40):
        L, k, V = 4, 1, 1
        tab = rng.normal(size=1 << L).astype(np.float32).astype(np.float64)
        s = rng.normal(size=6).astype(np.float32).astype(np.float64)
        st, c = viterbi.viterbi_f32(s, L, k, V, tab)
        bst, bc = viterbi.brute_force(s, L, k, V, tab)
        assert abs(_cost64(st, s, tab) - bc) <= 1e-5 * max(1.0, bc)      # optimal up to binary32 rounding
        assert abs(c - bc) <= 1e-5 * max(1.0, bc)
        for t in range(1, len(st)):                                       # a walk on the trellis
            assert (int(st[t]) >> k) == (int(st[t - 1]) & ((1 << (L - k)) - 1))


def test_f32_agrees_with_f64_dp_on_realistic_sequences():
    L, k, V = 16, 2, 1
    tab = codes.code_table("3inst", L)
    tab = tab / tab.std()
    rng = np.random.default_rng(12)
    S = rng.normal(size=(6, 64)).astype(np.float32)
    same = 0
    for s in S:
        st64, c64 = viterbi.viterbi(s.astype(np.float64), L, k, V, tab.astype(np.float32).astype(np.float64))
        st32, c32 = viterbi.viterbi_f32(s, L, k, V, tab)
        assert abs(c32 - c64) <= 1e-4 * c64
        assert abs(_cost64(st32, s.astype(np.float64), tab.astype(np.float32).astype(np.float64)) - c64) <= 1e-4 * c64
        same += int(np.array_equal(st32, st64))
    assert same >= 4                                                       # rounding-level ties only


def test_f32_tailbite_batch_is_tail_biting():
    L, k, V = 16, 2, 1
    tab = codes.code_table("3inst", L)
    tab = (tab / tab.std()).astype(np.float32)
    S = np.random.default_rng(13).normal(size=(3, 32)).astype(np.float32)
    st, cost = viterbi.tailbite_encode_f32_batch(S, L, k, V, tab)
    for w, c, s in zip(st, cost, S):
        # closure: the last state's bottom L-kV bits are the first state's top L-kV bits
        assert (int(w[0]) >> (k * V)) == (int(w[-1]) & ((1 << (L - k * V)) - 1))
        assert trellis.is_walk(w, L, k, V, tail_biting=True)
        # the reported cost is the squared error of the returned walk (binary32 rounding)
        assert abs(c - _cost64(w, s.astype(np.float64), tab.astype(np.float64))) <= 1e-4 * c


def test_f32_tailbite_batch_pinned_to_exact_optimum_and_f64_alg4():
    """Algorithm 4 in binary32 (the GPU quantizer's reference, reading R17) against things other
    than itself, on tiny trellises: the exact tail-biting optimum by brute force over every cyclic
    bit string (its cost is a lower bound Alg. 4 meets or exceeds), the float64 Alg. 4
    (pinned to Table 3 in test_oracle_viterbi.py) -- same walk whenever no two candidate costs lie
    within binary32 rounding of each other -- and P:348's seam rule checked on the walks: the
    constrained pass's first and last states share the overlap the rotated pass produced."""
    rng = np.random.default_rng(17)
    agree = 0
    for trial in range(30):
        L, k, V, T = 6, 2, 1, 8
        tab = rng.normal(size=1 << L).astype(np.float32)
        s = rng.normal(size=T).astype(np.float32)
        st, cost = viterbi.tailbite_encode_f32_batch(s[None, :], L, k, V, tab)
        st, cost = st[0], float(cost[0])
        _, best = viterbi.brute_force(s.astype(np.float64), L, k, V, tab.astype(np.float64), tail_biting=True)
        assert cost >= best * (1 - 1e-5) - 1e-6                              # never below the optimum
        assert trellis.is_walk(st, L, k, V, tail_biting=True)
        st64, c64 = viterbi.tailbite_encode(s.astype(np.float64), L, k, V, tab.astype(np.float64))
        assert abs(cost - c64) <= 1e-4 * max(1.0, c64)
        agree += int(np.array_equal(st, st64))
        # seam rule: the overlap O is the rotated walk's state at 1-indexed group T/2 (reading R3)
        srot = np.roll(s, T // 2)
        rot, _ = viterbi.viterbi_f32(srot, L, k, V, tab)
        O = int(rot[T // 2 - 1]) & ((1 << (L - k)) - 1)
        assert (int(st[0]) >> k) == O and (int(st[-1]) & ((1 << (L - k)) - 1)) == O
    assert agree >= 27
