// k_gemv_mma.cu -- fused trellis-decode GEMV with register-fed tensor-core MMA (impl 3).
//
// Each warp decodes straight into mma.sync.m16n8k16 A fragments and accumulates in registers:
// no shared memory, no TMEM, no cross-warp hand-off.  At batch <= 16 the contraction is <1%
// of the work; the bound is the integer decode (window extraction + LCG + LOP3, PAPER.md:
// 208-212, Alg. 1/2), and independent warps keep every SM sub-partition issuing.
//
// CTA = 4 warps walking a contiguous range of 128 x 128 cells (row-block major); warp w owns
// tile rows 2w and 2w+1 of every cell (they share the B fragments).  Thread 0 keeps a 4-deep
// ring of cells (packed stream + the cell's x~ columns) in flight with cp.async.bulk, so the
// decode reads shared memory instead of exposing global-load latency.  Fragment mapping for a 16 x 16 tile
// (rows permuted, K doubled for 3INST / 1MAD):
//   MMA row g (lane / 4)      <-> tile row 2g,   MMA row g + 8 <-> tile row 2g + 1
//   MMA 0 K-pair slots tig, tig+4 <-> columns 2 tig, 2 tig + 8   (tig = lane % 4)
//   MMA 1 K-pair slots tig, tig+4 <-> columns 2 tig + 1, 2 tig + 9
// so a lane's windows of one tile row sit at bit offsets 4 tig + {0, 2, 16, 18} of the row: two
// funnel shifts give all four, and tile rows 2g, 2g+1 share the words 2g .. 2g+2 (one 128-bit +
// one 64-bit load per tile pair).  For 3INST the LCG of the lower window is computed without
// masking it out, a x_lo + b = (a w + b) - (a x_hi) << 16, which moves work from the ALU to
// the FMA pipe.
// The A register of a K-doubled slot is the 3INST word (m1, m2) itself (B = x~ duplicated) or
// the 1MAD dp4a word half2(1024 + s, -1534); HYB uses the LUT pair (c0, c1) and plain x~.
// x~ arrives in fragment order (qtip RHT out_mode 3 / 4), so every lane loads its B fragment of
// a tile with one 128-bit (64-bit for HYB) shared-memory load.
// Partial sums per (cell, row) go to the workspace and are reduced in a fixed order.
#include "decode.cuh"
#include "internal.h"
#include "tc.cuh"

namespace qtip {
namespace {

constexpr int kMmaWarps = 4;
constexpr int kMmaStages = 4;                                    // bulk-copy ring depth (cells)

struct MmaArgs {
    const uint32_t* packed;
    Layout lay;
    CodeArgs ca;
    const uint32_t* lut;       // HYB: 2^Q words (c0 | c1 << 16)
    const uint32_t* xt;        // fragment-ordered x~ [8 NG][n_pad] (u32 per column, or per pair for HYB)
    int64_t xt_row_words;
    int B;
    int64_t rb0;
    int64_t units;             // cells in [rb0, rb1) x [0, n_kc), split evenly over the CTAs
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
__device__ __forceinline__ uint32_t umulhi_asm(uint32_t a, uint32_t b) {   // IMAD.HI: FMA pipe
    uint32_t r;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// Paper constants as compile-time immediates: IMAD / LOP3 with an immediate
// operand read one register less, which removes register-port dispatch stalls in the decode loop.
template <int CODE>
struct PaperLcg {
    static constexpr uint32_t a = (CODE == QTIP_CODE_1MAD) ? 34038481u : 89226354u;
    static constexpr uint32_t b = (CODE == QTIP_CODE_1MAD) ? 76625530u : 64248484u;
};

template <int CODE, bool kImm>
struct Lcg {
    uint32_t a, b;
    __device__ __forceinline__ Lcg(const CodeArgs& ca) : a(kImm ? PaperLcg<CODE>::a : ca.a), b(kImm ? PaperLcg<CODE>::b : ca.b) {}
    __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
        if constexpr (kImm) return x * PaperLcg<CODE>::a + PaperLcg<CODE>::b;
        else return x * a + b;
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
__device__ __forceinline__ void lcg_pair(uint32_t F, const Lcg<CODE, kImm>& lcg, uint32_t magic, uint32_t a_shl16,
                                         uint32_t& z_hi, uint32_t& z_lo) {
    const uint32_t x_hi = F >> 16;
    const uint32_t y_hi = lcg(x_hi);
    uint32_t y_lo;
    if constexpr (kLoOnFma) {
        y_lo = lcg(F);                                            // a F + b
        y_lo = x_hi * a_shl16 + y_lo;                             // - (a x_hi) << 16   (a_shl16 = -a << 16)
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

template <int K, int CODE, int NG, bool kImm>   // NG = batch groups of 8 (1 or 2); kImm = paper LCG constants
__global__ void __launch_bounds__(32 * kMmaWarps) gemv_mma_kernel(const MmaArgs args) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr bool kHyb = CODE == QTIP_CODE_HYB;
    constexpr int TW = 8 * K;
    constexpr uint32_t kCellBytes = 2048u * K;                      // packed stream of one cell
    constexpr uint32_t kXRowBytes = kHyb ? 256u : 512u;              // x~ of one cell, one batch row
    const uint32_t stage_bytes = kCellBytes + kXRowBytes * (8u * NG);   // x~ rows >= B stay zero
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);             // kMmaStages mbarriers
    uint8_t* stages = smem + 128;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, tig = lane & 3;
    const int n_kc = (int)args.lay.n_kc;
    const int64_t G = gridDim.x;
    const int64_t u0 = args.units * blockIdx.x / G, u1 = args.units * (blockIdx.x + 1) / G;
    const int nunits = (int)(u1 - u0);
    const CodeArgs ca = args.ca;
    const Lcg<CODE, kImm> lcg(ca);
    const uint32_t a_shl16 = (0u - lcg.a) << 16;

    if (threadIdx.x == 0) {
        for (int st = 0; st < kMmaStages; ++st) ptx::mbar_init(ptx::smem_u32(full + st), 1);
        ptx::fence_mbar_init();
    }
    for (int st = 0; st < kMmaStages; ++st) {                       // zero the padding batch rows once
        uint4* z = reinterpret_cast<uint4*>(stages + st * stage_bytes + kCellBytes + args.B * kXRowBytes);
        for (int i = threadIdx.x; i < (int)((8 * NG - args.B) * kXRowBytes / 16); i += 32 * kMmaWarps)
            z[i] = make_uint4(0u, 0u, 0u, 0u);
    }
    __syncthreads();
    auto issue = [&](int j) {                                        // thread 0: stage cell j of this CTA
        const int st = j % kMmaStages;
        const int64_t u = u0 + j;
        const int64_t RB = args.rb0 + u / n_kc, KC = u % n_kc;
        uint8_t* dst = stages + st * stage_bytes;
        const uint32_t bar = ptx::smem_u32(full + st);
        ptx::mbar_arrive_expect_tx(bar, kCellBytes + kXRowBytes * (uint32_t)args.B);
        ptx::bulk_g2s(ptx::smem_u32(dst), args.packed + (RB * n_kc + KC) * (int64_t)(kCellBytes / 4), kCellBytes, bar);
        for (int n = 0; n < args.B; ++n)
            ptx::bulk_g2s(ptx::smem_u32(dst + kCellBytes + n * kXRowBytes),
                          reinterpret_cast<const uint8_t*>(args.xt) + n * args.xt_row_words * 4 + KC * kXRowBytes,
                          kXRowBytes, bar);
    };
    // packed weights never depend on the previous kernel; x~ does
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    if (threadIdx.x == 0)
        for (int j = 0; j < min(nunits, kMmaStages); ++j) issue(j);

    for (int j = 0; j < nunits; ++j) {
        const int st = j % kMmaStages;
        const int64_t u = u0 + j;
        const int64_t RB = args.rb0 + u / n_kc, KC = u % n_kc;
        ptx::mbar_wait(ptx::smem_u32(full + st), (j / kMmaStages) & 1);
        const uint32_t* cell = reinterpret_cast<const uint32_t*>(stages + st * stage_bytes);
        const uint32_t* xs = reinterpret_cast<const uint32_t*>(stages + st * stage_bytes + kCellBytes);
        float acc[2][NG][4];
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int ng = 0; ng < NG; ++ng) acc[t][ng][0] = acc[t][ng][1] = acc[t][ng][2] = acc[t][ng][3] = 0.0f;
#pragma unroll
        for (int pp = 0; pp < kCellTileCols / 2; ++pp) {              // tile pair (2pp, 2pp+1)
            // ---- B fragments of both tile columns (shared by the warp's two tile rows)
            uint32_t bf[2][NG][4];
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const int J = 2 * pp + t;
#pragma unroll
                for (int ng = 0; ng < NG; ++ng) {
                    const int n = g + 8 * ng;                                // rows >= B are zero in smem
                    if constexpr (!kHyb) {
                        const uint4 v = *reinterpret_cast<const uint4*>(xs + n * 128 + J * 16 + tig * 4);
                        bf[t][ng][0] = v.x; bf[t][ng][1] = v.y; bf[t][ng][2] = v.z; bf[t][ng][3] = v.w;  // 2tig, 2tig+8, 2tig+1, 2tig+9
                    } else {
                        const uint2 v = *reinterpret_cast<const uint2*>(xs + n * 64 + J * 8 + tig * 2);
                        bf[t][ng][0] = v.x; bf[t][ng][1] = v.y; bf[t][ng][2] = bf[t][ng][3] = 0u;         // pairs tig, tig+4
                    }
                }
            }
#pragma unroll
            for (int tr = 0; tr < 2; ++tr) {
                const int I = 2 * warp + tr;
                const uint32_t* pw = cell + (I * 4 + pp) * TW * 2;          // word w of tile t at pw[2w + t]
                if constexpr (K == 2 && !kHyb) {
                    // tile rows 2g, 2g+1 use words 2g, 2g+1, 2g+2 (mod 16) of each tile
                    const uint4 w01 = *reinterpret_cast<const uint4*>(pw + 2 * (2 * g));
                    const uint2 w2 = *reinterpret_cast<const uint2*>(pw + 2 * ((2 * g + 2) & 15));
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        const uint32_t W0 = t ? w01.y : w01.x, W1 = t ? w01.w : w01.z, W2 = t ? w2.y : w2.x;
                        const uint32_t A0 = __funnelshift_l(W1, W0, 4 * tig);   // row 2g, from bit 4 tig
                        const uint32_t A1 = __funnelshift_l(W1, W0, 4 * tig + 2);
                        const uint32_t C0 = __funnelshift_l(W2, W1, 4 * tig);   // row 2g+1
                        const uint32_t C1 = __funnelshift_l(W2, W1, 4 * tig + 2);
                        uint32_t z00, z08, z01, z09, z10, z18, z11, z19;        // z<row><col offset>
                        constexpr bool kLoFma = CODE == QTIP_CODE_3INST;
                        lcg_pair<CODE, kLoFma, kImm>(A0, lcg, ca.magic, a_shl16, z00, z08);
                        lcg_pair<CODE, kLoFma, kImm>(A1, lcg, ca.magic, a_shl16, z01, z09);
                        lcg_pair<CODE, kLoFma, kImm>(C0, lcg, ca.magic, a_shl16, z10, z18);
                        lcg_pair<CODE, kLoFma, kImm>(C1, lcg, ca.magic, a_shl16, z11, z19);
#pragma unroll
                        for (int ng = 0; ng < NG; ++ng) {
                            hmma_16816(acc[tr][ng], z00, z10, z08, z18, bf[t][ng][0], bf[t][ng][1]);
                            hmma_16816(acc[tr][ng], z01, z11, z09, z19, bf[t][ng][2], bf[t][ng][3]);
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
                                zr[rr][0] = hyb_word(window_general(a0, a1, a2, off + tig * 2 * K), args.lut, ca.Q);
                                zr[rr][1] = hyb_word(window_general(a0, a1, a2, off + (tig + 4) * 2 * K), args.lut, ca.Q);
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
                            hmma_16816(acc[tr][ng], zr[0][0], zr[1][0], zr[0][1], zr[1][1], bf[t][ng][0], bf[t][ng][1]);
                            if constexpr (!kHyb)
                                hmma_16816(acc[tr][ng], zr[0][2], zr[1][2], zr[0][3], zr[1][3], bf[t][ng][2], bf[t][ng][3]);
                        }
                    }
                }
            }
        }
        __syncthreads();                                             // every warp is done with stage st
        if (threadIdx.x == 0 && j + kMmaStages < nunits) issue(j + kMmaStages);
        // ---- partial sums: acc[tr][ng] = D[MMA row g / g+8][batch 8 ng + 2 tig, + 1]
#pragma unroll
        for (int tr = 0; tr < 2; ++tr) {
            const int64_t row0 = RB * kCellRows + (2 * warp + tr) * kTile + 2 * g;   // tile row 2g (MMA row g)
#pragma unroll
            for (int ng = 0; ng < NG; ++ng) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int b = 8 * ng + 2 * tig + (e & 1);
                    const int64_t row = row0 + (e >> 1);                 // e >= 2: MMA row g + 8 = tile row 2g+1
                    if (b < args.B)
                        args.partial[(KC * args.B + b) * args.lay.m_pad + row] = acc[tr][ng][e] * args.code_factor;
                }
            }
        }
    }
}

template <int K, int CODE, int NG, bool kImm>
cudaError_t launch_mma_t(const MmaArgs& a, cudaStream_t s) {
    constexpr bool kHyb = CODE == QTIP_CODE_HYB;
    const size_t smem = 128 + (size_t)kMmaStages * (2048u * K + (kHyb ? 256u : 512u) * 8u * NG);
    auto kern = gemv_mma_kernel<K, CODE, NG, kImm>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * kMmaWarps, smem);
    const int64_t grid = std::min<int64_t>(a.units, (int64_t)std::max(1, per_sm) * num_sms());
    return launch_pdl(kern, dim3((unsigned)grid), dim3(32 * kMmaWarps), smem, s, a);
}

}  // namespace

bool gemv_mma_supported(const Layout& lay, int code, const CodeArgs& ca, int64_t B) {
    if (B < 1 || B > 16) return false;
    if (lay.k < 2 || lay.k > 4) return false;
    if (code == QTIP_CODE_HYB && ca.two_sign) return false;
    return true;
}

int gemv_mma_xt_mode(int code) { return code == QTIP_CODE_HYB ? 4 : 3; }
int gemv_mma_batch_pad(int64_t B) { return B > 8 ? 16 : 8; }

cudaError_t launch_gemv_mma(const Layout& lay, int code, const CodeArgs& ca, const void* packed, const uint16_t* lut,
                            const void* xt_frag, int64_t xt_row_words, int64_t B, int64_t rb0, int64_t rb1,
                            float* partial, cudaStream_t s) {
    MmaArgs a;
    a.packed = (const uint32_t*)packed;
    a.lay = lay;
    a.ca = ca;
    a.lut = (const uint32_t*)lut;
    a.xt = (const uint32_t*)xt_frag;
    a.xt_row_words = xt_row_words;
    a.B = (int)B;
    a.rb0 = rb0;
    a.code_factor = (code == QTIP_CODE_1MAD) ? 5.0f / 739.0f : 1.0f;
    a.partial = partial;
    a.units = (rb1 - rb0) * lay.n_kc;
    const bool ng2 = B > 8;
    const bool imm = code != QTIP_CODE_HYB && ca.a == (code == QTIP_CODE_1MAD ? 34038481u : 89226354u) &&
                     ca.b == (code == QTIP_CODE_1MAD ? 76625530u : 64248484u);
    cudaError_t e = cudaErrorInvalidValue;
#define QTIP_MMA_CASE(KK, CC)                                                                          \
    if (lay.k == KK && code == CC) {                                                                    \
        if (imm) e = ng2 ? launch_mma_t<KK, CC, 2, true>(a, s) : launch_mma_t<KK, CC, 1, true>(a, s);  \
        else e = ng2 ? launch_mma_t<KK, CC, 2, false>(a, s) : launch_mma_t<KK, CC, 1, false>(a, s);    \
    }
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
