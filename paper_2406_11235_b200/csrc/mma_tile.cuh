// mma_tile.cuh -- register-fed mma.sync decode of 16 x 16 trellis tiles (shared by the
// split-K GEMV k_gemv_mma.cu and the row-tile GEMV k_gemv_row.cu).
//
// Fragment mapping for a 16 x 16 tile (rows permuted, K doubled for 3INST / 1MAD):
//   MMA row g (lane / 4)      <-> tile row 2g,   MMA row g + 8 <-> tile row 2g + 1
//   MMA 0 K-pair slots tig, tig+4 <-> columns 2 tig, 2 tig + 8   (tig = lane % 4)
//   MMA 1 K-pair slots tig, tig+4 <-> columns 2 tig + 1, 2 tig + 9
// so a lane's windows of one tile row sit at bit offsets 4 tig + {0, 2, 16, 18} of the row: two
// funnel shifts give all four, and tile rows 2g, 2g+1 share the words 2g .. 2g+2 (one 128-bit +
// one 64-bit load per tile pair).  For 3INST the LCG of the lower window is computed without
// masking it out, a x_lo + b = (a w + b) - (a x_hi) << 16, which moves work from the ALU to
// the FMA pipe.  The A register of a K-doubled slot is the 3INST word (m1, m2) itself (B = x~
// duplicated) or the 1MAD dp4a word half2(1024 + s, -1534); HYB uses the LUT pair (c0, c1) and
// plain x~.  x~ arrives in fragment order (qtip RHT out_mode 3 / 4), so every lane loads its B
// fragment of a tile with one 128-bit (64-bit for HYB) shared-memory load.
#pragma once
#include "decode.cuh"

namespace qtip {
namespace mma {

__device__ __forceinline__ void hmma_16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                           uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}


// Paper constants as compile-time immediates: IMAD / LOP3 with an immediate
// operand read one register less, which removes register-port dispatch stalls in the decode loop.
template <int CODE>
struct PaperLcg {
    static constexpr uint32_t a = (CODE == QTIP_CODE_1MAD) ? 34038481u : 89226354u;
    static constexpr uint32_t b = (CODE == QTIP_CODE_1MAD) ? 76625530u : 64248484u;
};

// With kImm, a (and -a << 16) are immediates and b lives in a register the compiler cannot
// see through: an IMAD has one immediate slot, and otherwise ptxas spends it on b and
// rematerialises the other constant with an IMAD.MOV before every use.
__device__ __forceinline__ uint32_t opaque(uint32_t v) {
    uint32_t r;
    asm("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
    return r;
}

template <int CODE, bool kImm>
struct Lcg {
    uint32_t a, b, a_shl16;
    __device__ __forceinline__ Lcg(const CodeArgs& ca)
        : a(kImm ? PaperLcg<CODE>::a : ca.a), b(opaque(kImm ? PaperLcg<CODE>::b : ca.b)),
          a_shl16((0u - (kImm ? PaperLcg<CODE>::a : ca.a)) << 16) {}
    __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
        if constexpr (kImm) return x * PaperLcg<CODE>::a + b;
        else return x * a + b;
    }
    __device__ __forceinline__ uint32_t minus_hi(uint32_t x_hi, uint32_t y) const {   // y - (a x_hi) << 16
        if constexpr (kImm) return x_hi * ((0u - PaperLcg<CODE>::a) << 16) + y;
        else return x_hi * a_shl16 + y;
    }
};

template <int CODE>
__device__ __forceinline__ uint32_t code_from_lcg(uint32_t y, uint32_t magic) {
    if constexpr (CODE == QTIP_CODE_3INST) {
        uint32_t z;
        asm("lop3.b32 %0, %1, %2, %3, 0x6a;" : "=r"(z) : "r"(y), "r"(0x8FFF8FFFu), "r"(magic));
        return z;
    } else {
        return __dp4a(y, 0x01010101u, 0xE5FE6400u);      // half2(1024 + s, -1534)
    }
}

// Codes of the four windows of a funnel word F (top 16 bits and bottom 16 bits) ... here two
// words: windows hi(F) and lo(F).  y = a x + b on the FMA pipe; x_lo via LOP3 or via IMAD.
// Measured on B200 (scripts/alu_microbench.cu): IMAD, LOP3, SHF, PRMT, IDP.4A issue at 64
// lanes/clk/SM on their pipes, IMAD.HI at only 32 -- so the shift stays on the ALU pipe and the
// lower window goes to the FMA pipe for 3INST (2 IMAD instead of LOP3 + IMAD), which leaves
// 2 ALU + 1.5 FMA ops per weight.  1MAD's dp4a already loads the FMA pipe, so it keeps the LOP3.
template <int CODE, bool kLoOnFma, bool kImm>
__device__ __forceinline__ void lcg_pair(uint32_t F, const Lcg<CODE, kImm>& lcg, uint32_t magic,
                                         uint32_t& z_hi, uint32_t& z_lo) {
    const uint32_t x_hi = F >> 16;
    const uint32_t y_hi = lcg(x_hi);
    uint32_t y_lo;
    if constexpr (kLoOnFma) {
        y_lo = lcg.minus_hi(x_hi, lcg(F));                        // a F + b - (a x_hi) << 16
    } else {
        y_lo = lcg(F & 0xFFFFu);
    }
    z_hi = code_from_lcg<CODE>(y_hi, magic);
    z_lo = code_from_lcg<CODE>(y_lo, magic);
}

// HYB pair (c0 | c1 << 16) with the Alg. 3 sign flip of c1; x may carry garbage above bit 15.
__device__ __forceinline__ uint32_t hyb_word(uint32_t x, const uint32_t* __restrict__ lut, int Q) {
    const uint32_t h = x * x + x;
    uint32_t w = __ldg(lut + ((h >> (15 - Q)) & ((1u << Q) - 1u)));
    return w ^ ((h & 0x8000u) << 16);
}

// B fragments of tile column J of an x~ chunk in shared memory: batch row n at xs + n * row_words,
// tile J at + J * 16 (K-doubled codes: one u32 per column) or + J * 8 (HYB: one u32 per pair).
// Batch rows >= B read as zero (they only feed discarded accumulator columns).
template <int NG, bool kHyb>
__device__ __forceinline__ void load_bfrag(const uint32_t* xs, int row_words, int J, int g, int tig, int B,
                                           uint32_t (&bf)[NG][4]) {
#pragma unroll
    for (int ng = 0; ng < NG; ++ng) {
        const int n = g + 8 * ng;
        if constexpr (!kHyb) {
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if (n < B) v = *reinterpret_cast<const uint4*>(xs + n * row_words + J * 16 + tig * 4);
            bf[ng][0] = v.x; bf[ng][1] = v.y; bf[ng][2] = v.z; bf[ng][3] = v.w;   // 2tig, 2tig+8, 2tig+1, 2tig+9
        } else {
            uint2 v = make_uint2(0u, 0u);
            if (n < B) v = *reinterpret_cast<const uint2*>(xs + n * row_words + J * 8 + tig * 2);
            bf[ng][0] = v.x; bf[ng][1] = v.y; bf[ng][2] = bf[ng][3] = 0u;          // pairs tig, tig+4
        }
    }
}

// k = 2 3INST / 1MAD tile pair from preloaded words: w01 = words (2g, 2g+1) of both tiles
// (interleaved: .x/.y word 2g of tiles 0/1, .z/.w word 2g+1), w2 = word 2g+2 (mod 16) of both.
template <int CODE, int NG, bool kImm>
__device__ __forceinline__ void tile_pair_k2_words(const uint4 w01, const uint2 w2, const uint32_t (&bf)[2][NG][4],
                                                   float (&acc)[NG][4], int tig, const Lcg<CODE, kImm>& lcg,
                                                   const CodeArgs& ca) {
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const uint32_t W0 = t ? w01.y : w01.x, W1 = t ? w01.w : w01.z, W2 = t ? w2.y : w2.x;
        const uint32_t A0 = __funnelshift_l(W1, W0, 4 * tig);   // row 2g, from bit 4 tig
        const uint32_t A1 = __funnelshift_l(W1, W0, 4 * tig + 2);
        const uint32_t C0 = __funnelshift_l(W2, W1, 4 * tig);   // row 2g+1
        const uint32_t C1 = __funnelshift_l(W2, W1, 4 * tig + 2);
        uint32_t z00, z08, z01, z09, z10, z18, z11, z19;        // z<row><col offset>
        constexpr bool kLoFma = CODE == QTIP_CODE_3INST;
        lcg_pair<CODE, kLoFma, kImm>(A0, lcg, ca.magic, z00, z08);
        lcg_pair<CODE, kLoFma, kImm>(A1, lcg, ca.magic, z01, z09);
        lcg_pair<CODE, kLoFma, kImm>(C0, lcg, ca.magic, z10, z18);
        lcg_pair<CODE, kLoFma, kImm>(C1, lcg, ca.magic, z11, z19);
#pragma unroll
        for (int ng = 0; ng < NG; ++ng) {
            hmma_16816(acc[ng], z00, z10, z08, z18, bf[t][ng][0], bf[t][ng][1]);
            hmma_16816(acc[ng], z01, z11, z09, z19, bf[t][ng][2], bf[t][ng][3]);
        }
    }
}

// acc[ng] += W~(tiles t = 0, 1 of a tile pair) x~: pw = the pair's interleaved words (word w of
// tile t at pw[2w + t], TW = 8K words per tile), bf[t] the B fragments of tile t.
template <int K, int CODE, int NG, bool kImm>
__device__ __forceinline__ void tile_pair(const uint32_t* pw, const uint32_t (&bf)[2][NG][4], float (&acc)[NG][4],
                                          int g, int tig, const Lcg<CODE, kImm>& lcg, const CodeArgs& ca,
                                          const uint32_t* __restrict__ lut) {
    constexpr bool kHyb = CODE == QTIP_CODE_HYB;
    constexpr int TW = 8 * K;
    if constexpr (K == 2 && !kHyb) {
        // tile rows 2g, 2g+1 use words 2g, 2g+1, 2g+2 (mod 16) of each tile
        const uint4 w01 = *reinterpret_cast<const uint4*>(pw + 2 * (2 * g));
        const uint2 w2 = *reinterpret_cast<const uint2*>(pw + 2 * ((2 * g + 2) & 15));
        tile_pair_k2_words<CODE, NG, kImm>(w01, w2, bf, acc, tig, lcg, ca);
    } else {
        // general k: three words per tile row (rows 2g, 2g+1)
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            uint32_t zr[2][4];
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
                const int rho = 2 * g + rr;
                const int start = 16 * K * rho, w0 = start >> 5, off = start & 31;
                const uint32_t a0 = pw[2 * (w0 % TW) + t], a1 = pw[2 * ((w0 + 1) % TW) + t],
                               a2 = pw[2 * ((w0 + 2) % TW) + t];
                if constexpr (kHyb) {
                    // pair windows tig and tig + 4 of the row (kV = 2k bits per pair)
                    zr[rr][0] = hyb_word(window_general(a0, a1, a2, off + tig * 2 * K), lut, ca.Q);
                    zr[rr][1] = hyb_word(window_general(a0, a1, a2, off + (tig + 4) * 2 * K), lut, ca.Q);
                    zr[rr][2] = zr[rr][3] = 0u;
                } else {
                    zr[rr][0] = code_from_lcg<CODE>(window_general(a0, a1, a2, off + (2 * tig) * K) * lcg.a + lcg.b, ca.magic);
                    zr[rr][1] = code_from_lcg<CODE>(window_general(a0, a1, a2, off + (2 * tig + 8) * K) * lcg.a + lcg.b, ca.magic);
                    zr[rr][2] = code_from_lcg<CODE>(window_general(a0, a1, a2, off + (2 * tig + 1) * K) * lcg.a + lcg.b, ca.magic);
                    zr[rr][3] = code_from_lcg<CODE>(window_general(a0, a1, a2, off + (2 * tig + 9) * K) * lcg.a + lcg.b, ca.magic);
                }
            }
#pragma unroll
            for (int ng = 0; ng < NG; ++ng) {
                hmma_16816(acc[ng], zr[0][0], zr[1][0], zr[0][1], zr[1][1], bf[t][ng][0], bf[t][ng][1]);
                if constexpr (!kHyb)
                    hmma_16816(acc[ng], zr[0][2], zr[1][2], zr[0][3], zr[1][3], bf[t][ng][2], bf[t][ng][3]);
            }
        }
    }
}

// HYB, k = 4, V = 2, Q = 9 fast path (Alg. 3).  Lane (g, tig) owns tile rows
// 2g + rr (MMA rows g, g + 8) and the column pairs tig, tig + 4 of each row: pair windows at bit
// offsets 64 rho + 8 tig and + 32 of the tile stream.  With qa = (64 rho + 8 tig - 16) >> 5 and
// n = (64 rho + 8 tig - 16) & 31 (lane constants; qa = -1 wraps to the last word: those bits are
// above the window and HYB ignores them), x1 = funnel(W[qa+1], W[qa], n) and x2 = funnel(W[qa+2],
// W[qa+1], n) hold the windows in their low 16 bits -- one SHF per pair of weights, no zero fill:
// x^2 + x mod 2^16 depends on x mod 2^16 only.  The LUT lives in shared memory replicated 32x
// (entry e of replica r at word 32 e + r, conflict-free) as (c0 << 16) | c1, so the sign flip of
// Alg. 3 is a single LOP3 on bit 15 and the address is ((h + h) & 0xFF80) + 4 lane; the A words
// are then (c1, c0) per column pair and x~ comes with the pair halves swapped (RHT out_mode 5).
struct HybFastLane {
    int wa[2];          // word offsets (2 * word index, pair-interleaved) of W[qa], per row rr
    int wb[2], wc[2];   // W[qa + 1], W[qa + 2]
    uint32_t n;         // funnel amount (same for both rows)
};

__device__ __forceinline__ HybFastLane hyb_fast_lane(int g, int tig) {
    HybFastLane hl;
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
        const int s = 64 * (2 * g + rr) + 8 * tig - 16;
        const int q = s >> 5;                                  // arithmetic: -1 for s < 0
        hl.wa[rr] = 2 * ((q + 32) & 31);
        hl.wb[rr] = 2 * ((q + 33) & 31);
        hl.wc[rr] = 2 * ((q + 34) & 31);
        hl.n = (uint32_t)(s & 31);
    }
    return hl;
}

// kTwo: the two-sign variant: bit 31 of x^2 + x also flips c0 (bit 31 of the word);
// that bit depends on all of x, so the window is zero-filled first (one more LOP3).
template <bool kTwo = false>
__device__ __forceinline__ uint32_t hyb_fast_word(uint32_t x, uint32_t lut_lane) {
    if constexpr (kTwo) x &= 0xFFFFu;
    const uint32_t h = x * x + x;
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(lut_lane + ((h + h) & 0xFF80u)));
    uint32_t w;
    if constexpr (kTwo) asm("lop3.b32 %0, %1, %2, 0x80008000, 0x78;" : "=r"(w) : "r"(v), "r"(h));
    else asm("lop3.b32 %0, %1, %2, 0x8000, 0x78;" : "=r"(w) : "r"(v), "r"(h));      // v ^ (h & 0x8000)
    return w;
}

// acc += W~(tiles t = 0, 1 of a pair) x~ for the HYB k = 4 fast path; pw = the pair's words,
// lut_lane = shared-memory address of this lane's LUT replica, bf[t] from x~ mode 5.
template <int NG, bool kTwo = false>
__device__ __forceinline__ void tile_pair_hyb4(const uint32_t* pw, const uint32_t (&bf)[2][NG][4], float (&acc)[NG][4],
                                               const HybFastLane& hl, uint32_t lut_lane) {
    uint32_t z[2][2][2];                                       // [tile][row rr][pair: tig, tig + 4]
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
        const uint2 A = *reinterpret_cast<const uint2*>(pw + hl.wa[rr]);
        const uint2 Bw = *reinterpret_cast<const uint2*>(pw + hl.wb[rr]);
        const uint2 C = *reinterpret_cast<const uint2*>(pw + hl.wc[rr]);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const uint32_t a = t ? A.y : A.x, b = t ? Bw.y : Bw.x, c = t ? C.y : C.x;
            z[t][rr][0] = hyb_fast_word<kTwo>(__funnelshift_l(b, a, hl.n), lut_lane);
            z[t][rr][1] = hyb_fast_word<kTwo>(__funnelshift_l(c, b, hl.n), lut_lane);
        }
    }
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int ng = 0; ng < NG; ++ng)
            hmma_16816(acc[ng], z[t][0][0], z[t][1][0], z[t][0][1], z[t][1][1], bf[t][ng][0], bf[t][ng][1]);
}

// HYB fast path for k = 2, 3 (windows not byte-aligned, and the pair tig + 4 window is 8k bits
// after the pair tig one, so it may start in the same or the next word): per lane, row and window a
// word offset and funnel amount (lane constants), two LDS.64 (both tiles of the pair) per window.
template <int K>
struct HybFastLaneK {
    int w0[2][2];       // [row rr][window] pair-interleaved offset of W[q] (W[q + 1] is at w1)
    int w1[2][2];
    uint32_t n[2][2];
};

template <int K>
__device__ __forceinline__ HybFastLaneK<K> hyb_fast_lane_k(int g, int tig) {
    constexpr int TW = 8 * K;
    HybFastLaneK<K> hl;
#pragma unroll
    for (int rr = 0; rr < 2; ++rr)
#pragma unroll
        for (int w = 0; w < 2; ++w) {
            const int s = 16 * K * (2 * g + rr) + 2 * K * (tig + 4 * w) - 16;   // window start - 16
            const int q = s >> 5;                                                // -1 wraps: garbage bits
            hl.w0[rr][w] = 2 * ((q + TW) % TW);
            hl.w1[rr][w] = 2 * ((q + 1 + TW) % TW);
            hl.n[rr][w] = (uint32_t)(s & 31);
        }
    return hl;
}

template <int K, int NG, bool kTwo = false>
__device__ __forceinline__ void tile_pair_hyb_k(const uint32_t* pw, const uint32_t (&bf)[2][NG][4], float (&acc)[NG][4],
                                                const HybFastLaneK<K>& hl, uint32_t lut_lane) {
    uint32_t z[2][2][2];                                       // [tile][row rr][pair: tig, tig + 4]
#pragma unroll
    for (int rr = 0; rr < 2; ++rr)
#pragma unroll
        for (int w = 0; w < 2; ++w) {
            const uint2 A = *reinterpret_cast<const uint2*>(pw + hl.w0[rr][w]);
            const uint2 Bw = *reinterpret_cast<const uint2*>(pw + hl.w1[rr][w]);
            z[0][rr][w] = hyb_fast_word<kTwo>(__funnelshift_l(Bw.x, A.x, hl.n[rr][w]), lut_lane);
            z[1][rr][w] = hyb_fast_word<kTwo>(__funnelshift_l(Bw.y, A.y, hl.n[rr][w]), lut_lane);
        }
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int ng = 0; ng < NG; ++ng)
            hmma_16816(acc[ng], z[t][0][0], z[t][1][0], z[t][0][1], z[t][1][1], bf[t][ng][0], bf[t][ng][1]);
}

}  // namespace mma
}  // namespace qtip
