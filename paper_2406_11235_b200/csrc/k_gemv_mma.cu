// k_gemv_mma.cu -- fused trellis-decode GEMV with register-fed tensor-core MMA (impl 3).
//
// Each warp decodes straight into mma.sync.m16n8k16 A fragments and accumulates in registers:
// no shared memory, no TMEM, no cross-warp hand-off.  At batch <= 16 the contraction is 0.6%
// of the work; the bound is the integer decode (window extraction + LCG + LOP3, PAPER.md:
// 208-212, Alg. 1/2), and a per-warp pipeline keeps every SM sub-partition issuing.
//
// CTA = one row block (8 tile rows) x `cells` consecutive 128-column cells; warp w owns tile
// row w.  Fragment mapping for the 16 x 16 tile (rows permuted, K doubled for 3INST / 1MAD):
//   MMA row g (lane / 4)      <-> tile row 2g,   MMA row g + 8 <-> tile row 2g + 1
//   MMA 0 K-pair slots tig, tig+4 <-> columns 2 tig, 2 tig + 8   (tig = lane % 4)
//   MMA 1 K-pair slots tig, tig+4 <-> columns 2 tig + 1, 2 tig + 9
// so a lane's windows of one tile row sit at bit offsets 4 tig + {0, 2, 16, 18} of that row:
// two funnel shifts give all four (>> 16 and & 0xFFFF), and tile rows 2g, 2g+1 share the
// words 2g .. 2g+2 (one 128-bit + one 64-bit load per tile pair).
// The A register of a K-doubled slot is the 3INST word (m1, m2) itself (B = x~ duplicated) or
// the 1MAD dp4a word half2(1024 + s, -1534); HYB uses the LUT pair (c0, c1) and plain x~.
// Partial sums per (cell, row) go to the workspace and are reduced in a fixed order.
#include "decode.cuh"
#include "internal.h"
#include "tc.cuh"

namespace qtip {
namespace {

constexpr int kMmaWarps = 8;

struct MmaArgs {
    const uint32_t* packed;
    Layout lay;
    CodeArgs ca;
    const uint32_t* lut;       // HYB: 2^Q words (c0 | c1 << 16)
    const uint8_t* xt;         // compact binary16 x~ [B][n_pad]: u32 doubled (1MAD/3INST) or u16 (HYB)
    int64_t xt_row_bytes;
    int B;
    int64_t rb0;
    int cells;                 // cells per CTA along K
    float code_factor;
    float* partial;
};

__device__ __forceinline__ void hmma_16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                           uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint2 ldg_nc64(const void* p) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ uint4 ldg_nc128(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

template <int CODE>
__device__ __forceinline__ uint32_t code_word(uint32_t x, const CodeArgs& ca) {
    if constexpr (CODE == QTIP_CODE_3INST) return inst3_word(x, ca.a, ca.b, ca.magic);
    else return __dp4a(x * ca.a + ca.b, 0x01010101u, 0xE5FE6400u);   // half2(1024 + s, -1534)
}

// HYB pair (c0 | c1 << 16) with the Alg. 3 sign flip of c1; x may carry garbage above bit 15.
__device__ __forceinline__ uint32_t hyb_word(uint32_t x, const uint32_t* __restrict__ lut, int Q) {
    const uint32_t h = x * x + x;
    uint32_t w = __ldg(lut + ((h >> (15 - Q)) & ((1u << Q) - 1u)));
    return w ^ ((h & 0x8000u) << 16);
}

template <int K, int CODE, int NG>   // NG = batch groups of 8 (1 or 2)
__global__ void __launch_bounds__(32 * kMmaWarps) gemv_mma_kernel(const MmaArgs args) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, tig = lane & 3;
    const int n_kc = (int)args.lay.n_kc;
    const int splits = (n_kc + args.cells - 1) / args.cells;
    const int64_t RB = args.rb0 + blockIdx.x / splits;
    const int kc0 = (blockIdx.x % splits) * args.cells;
    const int kc1 = min(kc0 + args.cells, n_kc);
    const int I = warp;
    constexpr bool kHyb = CODE == QTIP_CODE_HYB;
    constexpr int TW = 8 * K;

    ptx::pdl_wait();
    ptx::pdl_launch_dependents();

    for (int kc = kc0; kc < kc1; ++kc) {
        const uint32_t* cell = args.packed + (RB * n_kc + kc) * args.lay.cell_words;
        float acc[NG][4];
#pragma unroll
        for (int ng = 0; ng < NG; ++ng) acc[ng][0] = acc[ng][1] = acc[ng][2] = acc[ng][3] = 0.0f;
#pragma unroll 2
        for (int p = 0; p < 4; ++p) {                           // tile pair (2p, 2p+1)
            const uint32_t* pw = cell + (I * 4 + p) * TW * 2;   // word w of tile t at pw[2w + t]
            // ---- B fragments for both tiles (batch column g, and g + 8 for NG = 2)
            uint32_t bf[2][NG][4];
#pragma unroll
            for (int t = 0; t < 2; ++t) {
#pragma unroll
                for (int ng = 0; ng < NG; ++ng) {
                    const int n = g + 8 * ng;
                    const int64_t col0 = (int64_t)kc * kCellCols + (2 * p + t) * kTile;
                    if (n < args.B) {
                        const uint8_t* xr = args.xt + n * args.xt_row_bytes;
                        if constexpr (!kHyb) {
                            const uint2 lo = __ldg(reinterpret_cast<const uint2*>(xr + 4 * (col0 + 2 * tig)));
                            const uint2 hi = __ldg(reinterpret_cast<const uint2*>(xr + 4 * (col0 + 2 * tig + 8)));
                            bf[t][ng][0] = lo.x; bf[t][ng][1] = hi.x;      // MMA 0: cols 2tig, 2tig+8
                            bf[t][ng][2] = lo.y; bf[t][ng][3] = hi.y;      // MMA 1: cols 2tig+1, 2tig+9
                        } else {
                            // one MMA per tile: K-pair slot tig <-> pair tig (cols 2tig, 2tig+1),
                            // slot tig+4 <-> pair tig+4
                            bf[t][ng][0] = __ldg(reinterpret_cast<const uint32_t*>(xr + 2 * (col0 + 2 * tig)));
                            bf[t][ng][1] = __ldg(reinterpret_cast<const uint32_t*>(xr + 2 * (col0 + 2 * tig + 8)));
                            bf[t][ng][2] = bf[t][ng][3] = 0u;
                        }
                    } else {
                        bf[t][ng][0] = bf[t][ng][1] = bf[t][ng][2] = bf[t][ng][3] = 0u;
                    }
                }
            }
            if constexpr (K == 2 && !kHyb) {
                // tile rows 2g, 2g+1 use words 2g, 2g+1, 2g+2 (mod 16) of each tile
                const uint4 w01 = ldg_nc128(pw + 2 * (2 * g));
                const uint2 w2 = ldg_nc64(pw + 2 * ((2 * g + 2) & 15));
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const uint32_t W0 = t ? w01.y : w01.x, W1 = t ? w01.w : w01.z, W2 = t ? w2.y : w2.x;
                    const uint32_t A0 = __funnelshift_l(W1, W0, 4 * tig);       // row 2g, from bit 4 tig
                    const uint32_t A1 = __funnelshift_l(W1, W0, 4 * tig + 2);
                    const uint32_t C0 = __funnelshift_l(W2, W1, 4 * tig);       // row 2g+1
                    const uint32_t C1 = __funnelshift_l(W2, W1, 4 * tig + 2);
                    const uint32_t z00 = code_word<CODE>(A0 >> 16, args.ca);      // row 2g,   col 2tig
                    const uint32_t z08 = code_word<CODE>(A0 & 0xFFFFu, args.ca);  // row 2g,   col 2tig+8
                    const uint32_t z01 = code_word<CODE>(A1 >> 16, args.ca);      // row 2g,   col 2tig+1
                    const uint32_t z09 = code_word<CODE>(A1 & 0xFFFFu, args.ca);  // row 2g,   col 2tig+9
                    const uint32_t z10 = code_word<CODE>(C0 >> 16, args.ca);      // row 2g+1, ...
                    const uint32_t z18 = code_word<CODE>(C0 & 0xFFFFu, args.ca);
                    const uint32_t z11 = code_word<CODE>(C1 >> 16, args.ca);
                    const uint32_t z19 = code_word<CODE>(C1 & 0xFFFFu, args.ca);
#pragma unroll
                    for (int ng = 0; ng < NG; ++ng) {
                        hmma_16816(acc[ng], z00, z10, z08, z18, bf[t][ng][0], bf[t][ng][1]);
                        hmma_16816(acc[ng], z01, z11, z09, z19, bf[t][ng][2], bf[t][ng][3]);
                    }
                }
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
                            zr[rr][0] = hyb_word(window_general(a0, a1, a2, off + tig * 2 * K), args.lut, args.ca.Q);
                            zr[rr][1] = hyb_word(window_general(a0, a1, a2, off + (tig + 4) * 2 * K), args.lut, args.ca.Q);
                            zr[rr][2] = zr[rr][3] = 0u;
                        } else {
                            zr[rr][0] = code_word<CODE>(window_general(a0, a1, a2, off + (2 * tig) * K), args.ca);
                            zr[rr][1] = code_word<CODE>(window_general(a0, a1, a2, off + (2 * tig + 8) * K), args.ca);
                            zr[rr][2] = code_word<CODE>(window_general(a0, a1, a2, off + (2 * tig + 1) * K), args.ca);
                            zr[rr][3] = code_word<CODE>(window_general(a0, a1, a2, off + (2 * tig + 9) * K), args.ca);
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
        // ---- partial sums: acc[ng] = D[row g / g+8][batch 8 ng + 2 tig, + 1]
        const int64_t row0 = RB * kCellRows + I * kTile + 2 * g;     // tile row 2g (MMA row g)
#pragma unroll
        for (int ng = 0; ng < NG; ++ng) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int b = 8 * ng + 2 * tig + (e & 1);
                const int64_t row = row0 + (e >> 1);                     // e >= 2: MMA row g + 8 = tile row 2g+1
                if (b < args.B) args.partial[((int64_t)kc * args.B + b) * args.lay.m_pad + row] = acc[ng][e] * args.code_factor;
            }
        }
    }
}

template <int K, int CODE, int NG>
cudaError_t launch_mma_t(const MmaArgs& a, int64_t nrb, cudaStream_t s) {
    const int splits = (int)((a.lay.n_kc + a.cells - 1) / a.cells);
    return launch_pdl(gemv_mma_kernel<K, CODE, NG>, dim3((unsigned)(nrb * splits)), dim3(32 * kMmaWarps), 0, s, a);
}

}  // namespace

bool gemv_mma_supported(const Layout& lay, int code, const CodeArgs& ca, int64_t B) {
    if (B < 1 || B > 16) return false;
    if (lay.k < 2 || lay.k > 4) return false;
    if (code == QTIP_CODE_HYB && ca.two_sign) return false;
    return true;
}

cudaError_t launch_gemv_mma(const Layout& lay, int code, const CodeArgs& ca, const void* packed, const uint16_t* lut,
                            const void* xt_compact, int64_t xt_row_bytes, int64_t B, int64_t rb0, int64_t rb1,
                            float* partial, cudaStream_t s) {
    MmaArgs a;
    a.packed = (const uint32_t*)packed;
    a.lay = lay;
    a.ca = ca;
    a.lut = (const uint32_t*)lut;
    a.xt = (const uint8_t*)xt_compact;
    a.xt_row_bytes = xt_row_bytes;
    a.B = (int)B;
    a.rb0 = rb0;
    a.code_factor = (code == QTIP_CODE_1MAD) ? 5.0f / 739.0f : 1.0f;
    a.partial = partial;
    const int64_t nrb = rb1 - rb0;
    // enough CTAs for ~8 per SM, each walking `cells` consecutive cells of its row block
    const int64_t target = 8LL * num_sms();
    int cells = 1;
    while (nrb * ((lay.n_kc + cells * 2 - 1) / (cells * 2)) >= target && cells < 16) cells *= 2;
    a.cells = cells;
    const bool ng2 = B > 8;
    cudaError_t e = cudaErrorInvalidValue;
#define QTIP_MMA_CASE(KK, CC) \
    if (lay.k == KK && code == CC) e = ng2 ? launch_mma_t<KK, CC, 2>(a, nrb, s) : launch_mma_t<KK, CC, 1>(a, nrb, s);
    QTIP_MMA_CASE(2, QTIP_CODE_3INST)
    QTIP_MMA_CASE(3, QTIP_CODE_3INST)
    QTIP_MMA_CASE(4, QTIP_CODE_3INST)
    QTIP_MMA_CASE(2, QTIP_CODE_1MAD)
    QTIP_MMA_CASE(3, QTIP_CODE_1MAD)
    QTIP_MMA_CASE(4, QTIP_CODE_1MAD)
    QTIP_MMA_CASE(2, QTIP_CODE_HYB)
    QTIP_MMA_CASE(3, QTIP_CODE_HYB)
    QTIP_MMA_CASE(4, QTIP_CODE_HYB)
#undef QTIP_MMA_CASE
    count_launch(1);
    return e;
}

}  // namespace qtip
