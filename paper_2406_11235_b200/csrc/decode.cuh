// decode.cuh -- per-thread trellis window extraction and code evaluation (sm_100a).
//
// A thread owns one output row r of a tile; the row's 16 weights are the contiguous
// sequence positions 16r .. 16r+15 (row-major scan), so its windows are
// the L = 16-bit windows at bit offsets 16kr + q*kV of the tile stream (PAPER.md:208-212,
// bitshift trellis: "obtaining the next compressed group ... only requires bitshifting").
// Words are big-endian (stream bit 32w = bit 31 of word w) and wrap mod 8k words
// (tail-biting).
#pragma once
#include "common.cuh"

namespace qtip {

// ------------------------------------------------------------------ windows
// k = 2, V = 1: A = word r, B = word r+1 (mod 16) hold stream bits [32r, 32r+64) of the tile;
// window q (q = 0..15) is bits [2q, 2q+16) of A:B, zero-extended (1MAD/3INST need the
// zero fill: the LCG's upper half depends on every bit of x).
// Four phase copies P = (A:B) << 2p and four cross copies R = (A:B) << (24+2p); each
// window is then one byte-permute or one shift: 23 ALU ops for 16 windows.
__device__ __forceinline__ void windows_k2v1(uint32_t A, uint32_t B, uint32_t x[16]) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const uint32_t P = (p == 0) ? A : __funnelshift_l(B, A, 2 * p);   // bits [2p, 2p+32)
        const uint32_t R = __funnelshift_l(B, A, 24 + 2 * p);            // bits [24+2p, 56+2p)
        x[p] = P >> 16;                           // bits [2p,    2p+16)
        x[p + 4] = __byte_perm(P, 0u, 0x4421);    // bits [2p+8,  2p+24)
        x[p + 8] = __byte_perm(P, 0u, 0x4410);    // bits [2p+16, 2p+32)
        x[p + 12] = R >> 16;                      // bits [2p+24, 2p+40)
    }
}

// k = 4, V = 2: A, B, C = words 2r, 2r+1, 2r+2 (mod 32); pair-window q (q = 0..7) is bits
// [8q, 8q+16) of A:B:C.  HYB only reads hash bits 0..15, and x*x + x mod 2^16 depends only
// on x mod 2^16, so the window may carry garbage above bit 15: 6 ops for 8 windows.
__device__ __forceinline__ void windows_k4v2_dirty(uint32_t A, uint32_t B, uint32_t C, uint32_t x[8]) {
    x[0] = A >> 16;
    x[1] = A >> 8;
    x[2] = A;
    x[3] = __funnelshift_l(B, A, 8);
    x[4] = B >> 16;
    x[5] = B >> 8;
    x[6] = B;
    x[7] = __funnelshift_l(C, B, 8);
}

// General window: bits [pos, pos+16) of the 96-bit big-endian span W0:W1:W2, pos < 80.
__device__ __forceinline__ uint32_t window_general(uint32_t W0, uint32_t W1, uint32_t W2, int pos) {
    const uint64_t hi = (pos < 32) ? (((uint64_t)W0 << 32) | W1) : (((uint64_t)W1 << 32) | W2);
    const int p = pos & 31;
    return (uint32_t)(hi >> (48 - p)) & 0xFFFFu;
}

// ------------------------------------------------------------------ codes
// 3INST (Alg. 2): z = ((a x + b) & 0x8FFF8FFF) ^ (m << 16 | m).
// One IMAD and one LOP3 (both constants in registers so ptxas fuses AND + XOR).
__device__ __forceinline__ uint32_t inst3_word(uint32_t x, uint32_t a, uint32_t b, uint32_t magic) {
    const uint32_t y = x * a + b;
    uint32_t z;
    asm("lop3.b32 %0, %1, %2, %3, 0x6a;" : "=r"(z) : "r"(y), "r"(0x8FFF8FFFu), "r"(magic));
    return z;
}

// binary16 RNE of m1 + m2 (the footnote of PAPER.md:265: summed as two FP16s).
__device__ __forceinline__ __half inst3_value(uint32_t z) {
    return __hadd(__ushort_as_half((unsigned short)(z & 0xFFFFu)), __ushort_as_half((unsigned short)(z >> 16)));
}

// 1MAD (Alg. 1): s = bytesum(a x + b) via the unsigned dp4a.
__device__ __forceinline__ uint32_t onemad_sum(uint32_t x, uint32_t a, uint32_t b) {
    const uint32_t y = x * a + b;
    return __dp4a(y, 0x01010101u, 0u);
}

// binary16 RNE of (s - 510)/147.8: fp32 (s-510) * fl32(5/739) then one RNE conversion; equal
// to the correctly rounded value for all 1021 sums (checked exhaustively in the tests).
__device__ __forceinline__ __half onemad_value(uint32_t s) {
    return __float2half_rn(__fmul_rn((float)((int)s - 510), 5.0f / 739.0f));
}

// HYB (Alg. 3): h = x*x + x; index bits (15-Q)..14; sign from bit 15
// (and bit 31 with two_sign, which needs a zero-filled x).  LUT in global memory as
// (c0, c1) binary16 pairs; the flip of bit 15 of the word (c0 << 16 | c1) negates c1.
__device__ __forceinline__ void hyb_values(uint32_t x, const uint16_t* __restrict__ lut, int Q, int two_sign,
                                           uint16_t& c0, uint16_t& c1) {
    const uint32_t h = x * x + x;
    const uint32_t idx = (h >> (15 - Q)) & ((1u << Q) - 1u);
    c0 = lut[2 * idx];
    c1 = lut[2 * idx + 1];
    c1 ^= (uint16_t)(h & 0x8000u);
    if (two_sign) c0 ^= (uint16_t)((h >> 16) & 0x8000u);
}

}  // namespace qtip
