"""Pins for oracle.codes: golden values derived by hand / exact integer evaluation, closed-form
moments, the paper's counting claims, symmetry and neighbour correlation (Fig. 3)."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import codes


# ---------------------------------------------------------------- binary16 rounding
def test_fp16_rne_known_patterns():
    assert codes.fp16_rne(Fraction(1)) == 0x3C00
    assert codes.fp16_rne(Fraction(-2)) == 0xC000
    assert codes.fp16_rne(Fraction(65504)) == 0x7BFF
    assert codes.fp16_rne(Fraction(65520)) == 0x7C00                     # rounds to inf
    assert codes.fp16_rne(Fraction(1, 1 << 24)) == 0x0001                # smallest subnormal
    assert codes.fp16_rne(Fraction(1, 1 << 14)) == 0x0400                # smallest normal
    assert codes.fp16_rne(1 + Fraction(1, 2048)) == 0x3C00               # tie -> even (down)
    assert codes.fp16_rne(1 + Fraction(3, 2048)) == 0x3C02               # tie -> even (up)
    assert codes.fp16_rne(Fraction(1, 10)) == 0x2E66                     # 0.1 -> 0.0999755859375
    assert codes.fp16_rne(Fraction("0.922")) == 0x3B60                   # P:267 m = 0.922 -> 0.921875
    for b in [0x3C00, 0x2E66, 0xBD02, 0x0001, 0x7BFF, 0x8400]:
        assert codes.fp16_rne(codes.fp16_value(b)) == b


# ---------------------------------------------------------------- 1MAD (Alg. 1)
def test_1mad_golden():
    # x = 0: LCG gives b = 76625530 = 0x0491367A; bytes 0x04+0x91+0x36+0x7A = 4+145+54+122 = 325;
    # (325-510)/147.8 = -1.25169... -> binary16 -1.251953125 = 0xBD02   (hand evaluation of Alg. 1)
    assert codes.lcg(0, codes.A_1MAD, codes.B_1MAD) == 0x0491367A
    assert int(codes.byte_sum(0x0491367A)) == 325
    assert int(codes.decode_1mad(0)) == 0xBD02
    # x = 1: a + b = 34038481 + 76625530 = 110664011 = 0x0698994B; 6+152+153+75 = 386
    assert codes.lcg(1, codes.A_1MAD, codes.B_1MAD) == 0x0698994B
    assert int(codes.byte_sum(0x0698994B)) == 386
    assert int(codes.decode_1mad(1)) == 0xBAB6
    # further values from an independent big-integer evaluation (SURVEY §8(c) pins table)
    assert [int(codes.byte_sum(codes.lcg(x, codes.A_1MAD, codes.B_1MAD))) for x in (2, 0x1234, 0xFFFF)] == [447, 734, 571]
    assert [int(codes.decode_1mad(x)) for x in (2, 0x1234, 0xFFFF)] == [0xB6D2, 0x3E10, 0x369B]
    # SPEC S:153-154 trivial cases: a = b = 0 -> sum 0 -> (0-510)/147.8; b = 0x00FFFF00 -> 0.0
    assert int(codes.decode_1mad(0, a=0, b=0)) == codes.fp16_rne(Fraction(-510) / Fraction("147.8"))
    assert int(codes.decode_1mad(0, a=0, b=0x00FFFF00)) == 0


def test_1mad_rounding_is_correct_rne_of_exact_rational():
    s = np.arange(1021)
    got = codes.onemad_value_from_sum(s)
    for t in range(0, 1021):
        exact = Fraction(t - 510) / Fraction("147.8")
        v = codes.fp16_value(int(got[t]))
        # RNE error <= half an ulp <= 2^-11 |exact| (all values are normal binary16 here)
        assert abs(v - exact) <= abs(exact) / 2048


def test_1mad_moments_and_support():
    """Sum of 4 uniform bytes: mean 4*127.5 = 510, variance 4*(256^2-1)/12 -> std 147.80;
    the LCG over all 2^16 states should give ~N(0,1); at most 2^10 representable values."""
    assert abs(np.sqrt(4 * (256 ** 2 - 1) / 12) - 147.8) < 0.01
    xs = np.arange(1 << 16)
    sums = codes.byte_sum(codes.lcg(xs, codes.A_1MAD, codes.B_1MAD))
    assert len(np.unique(sums)) <= 1 << 10
    v = codes.code_table("1mad", 16)
    assert abs(v.mean()) < 0.01
    assert 0.98 < v.var() < 1.02


# ---------------------------------------------------------------- 3INST (Alg. 2)
def test_3inst_golden():
    assert codes.magic_word_3inst() == 0x3B603B60          # P:290, m = fp16(0.922) = 0x3B60
    # x = 0: y = b = 64248484 = 0x03D45AA4; & 0x8FFF8FFF = 0x03D40AA4; ^ 0x3B603B60 = 0x38B431C4
    z, tot, bits = codes.decode_3inst_exact(0)
    assert z == 0x38B431C4
    assert tot == codes.fp16_value(0x31C4) + codes.fp16_value(0x38B4)
    assert bits == 0x3A25 and int(codes.decode_3inst(0)) == 0x3A25        # 0.76806640625, exact
    z, tot, bits = codes.decode_3inst_exact(1)
    assert z == 0x3245BC76 and bits == 0xBB5B                               # exact -0.9193115234375 rounds
    assert tot == Fraction("-0.9193115234375")
    table = {2: (0x351738E8, 0x3B74), 0x1234: (0xB841BEAC, 0xC066), 0xFFFF: (0x3194B552, 0xB110)}
    for x, (zz, bb) in table.items():
        z, _, bits = codes.decode_3inst_exact(x)
        assert (z, bits) == (zz, bb)
        assert int(codes.decode_3inst(x)) == bb
    # LCG word 0 -> m + m = 1.84375 ; both sign bits -> -1.84375
    assert codes.fp16_value(int(codes.decode_3inst(0, a=0, b=0))) == Fraction(59, 32)
    assert codes.fp16_value(int(codes.decode_3inst(0, a=0, b=0x80008000))) == -Fraction(59, 32)


def test_3inst_field_structure_and_variance():
    """the mask keeps sign, the bottom two exponent bits and the mantissa; XOR with m
    fixes exponent bits 14..12 to 011 -> |m_i| in [2^-3, 2).  Variance of m1 + m2 for
    independent uniform fields (closed form over the 2^13 free patterns) vs all 2^16 states."""
    m1, m2 = codes.inst3_halves(np.arange(1 << 16))
    v1 = np.abs(codes.f16_to_f64(m1))
    assert v1.min() >= 0.125 and v1.max() < 2.0
    # closed form: enumerate the free bits (sign, e1 e0, mantissa) of one half
    vals = []
    for e in range(4):
        for mant in range(1024):
            bits = (0b011 << 12) | ((e ^ 0b10) << 10) | (mant ^ 0x360)      # XOR with 0x3B60's low fields
            vals.append(float(codes.fp16_value(bits)))
    e_m2 = np.mean(np.square(vals))                                         # sign symmetric: mean 0
    analytic_var = 2 * e_m2
    assert abs(analytic_var - 1.5495) < 1e-3
    t = codes.code_table("3inst", 16)
    assert abs(t.mean()) < 0.01
    assert abs(t.var() - analytic_var) < 0.01          # NOT ~1: SPEC S:223's gate is wrong (reading R9)


def test_3inst_sign_symmetry():
    rng = np.random.default_rng(3)
    for x in rng.integers(0, 1 << 16, 50):
        z, tot, _ = codes.decode_3inst_exact(int(x))
        zf = z ^ 0x80008000
        assert codes.fp16_value(zf & 0xFFFF) + codes.fp16_value(zf >> 16) == -tot


# ---------------------------------------------------------------- HYB (Alg. 3)
def test_hyb_hash_golden():
    # x = 3 -> 3*3 + 3 = 12 -> index (12 >> 6) & 511 = 0
    assert int(codes.hyb_hash(3)) == 12 and int(codes.hyb_index(12, 9)) == 0
    h = int(codes.hyb_hash(0x1234))
    assert h == 0x1234 * 0x1234 + 0x1234 == 0x014B6CC4
    assert int(codes.hyb_index(h, 9)) == (0x6CC4 >> 6) & 511 == 435 and (h >> 15) & 1 == 0
    h = int(codes.hyb_hash(0xFFFF))
    assert h == 0xFFFF0000                    # 0xFFFF^2 + 0xFFFF = 0xFFFF * 0x10000
    assert int(codes.hyb_index(h, 9)) == 0 and (h >> 15) & 1 == 0 and (h >> 31) & 1 == 1


def test_hyb_counting_claims():
    """an L-bit word maps to one of 2^{Q+1} 2-D vectors; at L=16 each index is hit
    exactly 2^{16-Q} times (x^2+x is 2-to-1 onto even residues)."""
    Q = 9
    h = codes.hyb_hash(np.arange(1 << 16))
    idx = codes.hyb_index(h, Q)
    assert (np.bincount(idx, minlength=1 << Q) == 1 << (16 - Q)).all()
    sign = (h >> np.uint64(15)) & np.uint64(1)
    assert len(set(zip(idx.tolist(), sign.tolist()))) == 1 << (Q + 1)
    assert (1 << Q) * 2 * 2 == 2048                                  # Q=9 -> 2 KiB LUT


def test_hyb_sign_flips_second_entry():
    lut = np.array([[0x3C00, 0x4000]] * 512, dtype=np.uint16)      # c0 = 1.0, c1 = 2.0
    xs = np.arange(1 << 16)
    out = codes.decode_hyb(xs, lut, 9)
    h = codes.hyb_hash(xs)
    flip = ((h >> np.uint64(15)) & np.uint64(1)).astype(bool)
    assert (out[:, 0] == 0x3C00).all()
    assert (out[flip, 1] == 0xC000).all() and (out[~flip, 1] == 0x4000).all()
    two = codes.decode_hyb(xs, lut, 9, two_sign=True)                # bit 31 flips the other entry
    f31 = ((h >> np.uint64(31)) & np.uint64(1)).astype(bool)
    assert (two[f31, 0] == 0xBC00).all() and (two[~f31, 0] == 0x3C00).all()


def test_kmeans_lut_basic():
    c0 = codes.f16_to_f64(codes.kmeans_lut(0, seed=1, n_samples=1 << 16, iters=5))
    assert np.abs(c0).max() < 0.05                                   # mean of N(0,I)
    c1 = codes.f16_to_f64(codes.kmeans_lut(1, seed=1, n_samples=1 << 16, iters=30))
    assert np.abs(c1[0] + c1[1]).max() < 0.05                        # symmetric pair
    lut = codes.kmeans_lut(6, seed=2, n_samples=1 << 15, iters=20)
    assert lut.shape == (64, 2) and np.isfinite(codes.f16_to_f64(lut)).all()


def test_distortion_rate_bound():
    assert codes.distortion_rate_bound(2) == 0.0625                  # Table 1 D_R "0.063"
    assert codes.distortion_rate_bound(0) == 1.0 and codes.distortion_rate_bound(4) == 0.00390625


def test_neighbour_correlation_fig3():
    """Fig. 3: the identity ramp is strongly correlated along edges; 1MAD slightly; 3INST ~ random."""
    L = 16
    ramp = np.arange(1 << L, dtype=np.float64)
    for k in (1, 2, 3):
        assert abs(codes.neighbor_correlation(ramp, L, k) - 2.0 ** (-k)) < 0.01
    assert abs(codes.neighbor_correlation(codes.code_table("3inst", L), L, 2)) < 0.01
    r1 = codes.neighbor_correlation(codes.code_table("1mad", L), L, 2)
    assert 0.001 < abs(r1) < 0.05
    assert codes.neighbor_correlation(np.ones(1 << L), L, 2) == 0.0
