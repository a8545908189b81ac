// umma_decode.cuh -- thread-per-row trellis decode of a tile pair into the A operand of a
// tcgen05.mma held in TMEM (shared by the stream-K GEMV, k_umma.cu, and the chain kernel, k_chain.cu).
//
// Thread = one row rho (0..15) of both tiles of a column pair, i.e. one TMEM lane: it reads its row's
// stream words from the cell in shared memory, extracts the 16 trellis windows of each tile row
// (tail-biting wrap P:325-328), evaluates the code (Alg. 1-3) and writes
// 16 binary16 weights per tile (two per 32-bit TMEM column) with tcgen05.st.
#pragma once
#include "decode.cuh"
#include "mma_tile.cuh"
#include "tc.cuh"

namespace qtip {
namespace udec {

// binary16 sums of the two halves of za and of zb, packed (lo: za, hi: zb), RNE.  Two scalar half adds
// whose operands are half-selectors of one register each (HADD2 Rz.H0_H0, Rz.H1_H1) and one PRMT to
// pack: 1 FMA-pipe + 0.5 ALU instruction per weight, instead of two PRMT transposes + one HADD2
// (1 ALU + 0.5 FMA) -- the ALU pipe is the 3INST decode's binding one (DESIGN 5.5)
__device__ __forceinline__ uint32_t pair_sum(uint32_t za, uint32_t zb) {
    uint32_t r;
    asm("{\n\t.reg .f16 a0, a1, b0, b1, s0, s1;\n\t"
        "mov.b32 {a0, a1}, %1;\n\t"
        "mov.b32 {b0, b1}, %2;\n\t"
        "add.rn.f16 s0, a0, a1;\n\t"
        "add.rn.f16 s1, b0, b1;\n\t"
        "mov.b32 %0, {s0, s1};\n\t}"
        : "=r"(r) : "r"(za), "r"(zb));
    return r;
}

// ---------------------------------------------------------------------------------------- decode
// This thread's row rho of the tile pair at pw (word w of tile t at pw[2w + t]) -> the A operand of
// both tiles (binary16 weights, columns 2i, 2i+1 in TMEM column i), at TMEM columns ta (tile 0) and
// ta + 8 (tile 1).
template <int K, int CODE, bool kImm>
__device__ __forceinline__ void decode_pair(const uint32_t* __restrict__ pw, int rho, const CodeArgs& ca,
                                            uint32_t lut_lane, uint32_t ta) {
    constexpr bool kHyb = CODE == QTIP_CODE_HYB;
    constexpr int TW = 8 * K;
    if constexpr (K == 2 && !kHyb) {
        const uint2 A = *reinterpret_cast<const uint2*>(pw + 2 * rho);
        const uint2 Bw = *reinterpret_cast<const uint2*>(pw + 2 * ((rho + 1) & 15));
        const mma::Lcg<CODE, kImm> lcg(ca);
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
            const uint32_t a = tt ? A.y : A.x, b = tt ? Bw.y : Bw.x;
            uint32_t z[16], o[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                // F_q = bits [2q, 2q + 32) of the row: windows q (high half) and q + 8 (low half)
                const uint32_t F = q ? __funnelshift_l(b, a, 2 * q) : a;
                mma::lcg_pair<CODE, CODE == QTIP_CODE_3INST, kImm>(F, lcg, ca.magic, z[q], z[q + 8]);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) o[i] = pair_sum(z[2 * i], z[2 * i + 1]);
            ptx::tmem_st8(ta + tt * 8, o);
        }
    } else if constexpr (K == 4 && kHyb) {
        const uint4 AB = *reinterpret_cast<const uint4*>(pw + 4 * rho);      // words 2 rho, 2 rho + 1 of both tiles
        const uint2 Cw = *reinterpret_cast<const uint2*>(pw + 2 * ((2 * rho + 2) & 31));
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
            uint32_t x[8], z[8];
            windows_k4v2_dirty(tt ? AB.y : AB.x, tt ? AB.w : AB.z, tt ? Cw.y : Cw.x, x);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t h = x[q] * x[q] + x[q];                         // Alg. 3 hash (bits 0..15 exact)
                const uint32_t off = (h & 0xFFC0u) * 2u + lut_lane;             // entry (idx | sign << 9) * 128 + lane
                asm volatile("ld.shared.b32 %0, [%1];" : "=r"(z[q]) : "r"(off));
            }
            ptx::tmem_st8(ta + tt * 8, z);
        }
    } else {
        // general k (3INST / 1MAD k = 3, 4; HYB k = 2, 3): windows from three words of the tile row
        const int start = 16 * K * rho, w0 = start >> 5, off = start & 31;
        const uint2 W0 = *reinterpret_cast<const uint2*>(pw + 2 * (w0 % TW));
        const uint2 W1 = *reinterpret_cast<const uint2*>(pw + 2 * ((w0 + 1) % TW));
        const uint2 W2 = *reinterpret_cast<const uint2*>(pw + 2 * ((w0 + 2) % TW));
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
            const uint32_t a0 = tt ? W0.y : W0.x, a1 = tt ? W1.y : W1.x, a2 = tt ? W2.y : W2.x;
            uint32_t o[8];
            if constexpr (kHyb) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint32_t x = window_general(a0, a1, a2, off + q * 2 * K);
                    const uint32_t h = x * x + x;
                    const uint32_t ad = (h & 0xFFC0u) * 2u + lut_lane;
                    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(o[q]) : "r"(ad));
                }
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    uint32_t zz[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const uint32_t x = window_general(a0, a1, a2, off + (2 * i + e) * K);
                        zz[e] = mma::code_from_lcg<CODE>(x * ca.a + ca.b, ca.magic);
                    }
                    o[i] = pair_sum(zz[0], zz[1]);
                }
            }
            ptx::tmem_st8(ta + tt * 8, o);
        }
    }
}

}  // namespace udec
}  // namespace qtip
