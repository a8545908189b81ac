// k_gemv_tc.cu -- fused trellis-decode GEMV/GEMM on the 5th-generation tensor cores (impl 2).
//
// Work unit = one 128 x 128 cell (8 x 8 tiles, PAPER.md:389-390 T_x = T_y = 16).  A persistent
// CTA per SM owns a contiguous range of cells and runs four independent row-block pipelines
// ("groups") that share one TMA producer warp and one MMA-issuing warp:
//
//   warp 0      producer: cp.async.bulk of each cell's packed stream (2048k bytes) into an
//               8-slot shared-memory ring (mbarrier complete_tx).
//   warp 1      allocates 512 TMEM columns; one lane issues tcgen05.mma (kind::f16, M=128,
//               N=16, K=16, A from TMEM, B from shared memory) and tcgen05.commit.
//   warps 2-17  decoders, 4 groups x 4 warps.  Thread (quadrant q, lane l) owns output row
//               R = 32q + l of its group's cell: it reads the row's words of two tiles with
//               64/128-bit LDS, extracts the 16 contiguous trellis windows of each tile row
//               (PAPER.md:208-212), evaluates the code (1MAD/3INST/HYB, Alg. 1-3) and stores
//               the A operand straight into its own TMEM lane with tcgen05.st.
//
// A-operand encodings (one 32-bit TMEM column = two K elements):
//   3INST  the masked/XORed LCG word (m1, m2) itself; B holds x~ duplicated, so the MMA forms
//          m1 x + m2 x exactly ("K-doubling"): no fp16 add, no data movement.
//   1MAD   dp4a(y, 0x01010101, 0xE5FE6400) = half2(1024 + s, -1534); with x~ duplicated the
//          MMA forms (s - 510) x exactly; 1/147.8 is applied to the partial sums.
//   HYB    the looked-up LUT pair (c0, c1) with the sign of Alg. 3 already folded into a
//          2^(Q+1)-entry, 32-way replicated shared-memory table (conflict-free LDS).
// Partial sums per (cell column, row) go to the workspace and are reduced in fixed order.
#include "decode.cuh"
#include "internal.h"
#include "tc.cuh"

namespace qtip {
namespace {

constexpr int kGroups = 4;
constexpr int kDecWarps = 4 * kGroups;
constexpr int kThreads = 32 * (2 + kDecWarps);   // 576
constexpr int kSlots = 8;
constexpr int kHyBLutQ = 9;
constexpr uint32_t kLutBytes = (1u << (kHyBLutQ + 1)) * 128u;   // 2^(Q+1) entries x 32 replicas x 4 B
constexpr int kN = 16;                                          // UMMA N (batch padded)

struct TcArgs {
    const uint32_t* packed;
    Layout lay;
    CodeArgs ca;
    const uint32_t* lut;       // HYB: 2^Q words, low half c0, high half c1
    const uint8_t* xt;         // compact fp16 x~: [B][n_pad] (u32 doubled or u16 plain)
    int64_t xt_row_bytes;
    int B;
    int64_t rb0;
    int64_t units;             // cells in [rb0, rb1) x [0, n_kc)
    float code_factor;
    float* partial;
};

template <int K, int CODE>
struct Cfg {
    static constexpr bool kHyb = CODE == QTIP_CODE_HYB;
    static constexpr int kColsPerTile = kHyb ? 8 : 16;          // TMEM columns of one tile row
    static constexpr int kMmaPerTile = kHyb ? 1 : 2;            // K = 16 per MMA
    static constexpr int kMmaPerUnit = 8 * kMmaPerTile;
    static constexpr uint32_t kUnitBytes = 2048u * K;
    static constexpr int kXtVecs = kHyb ? 16 : 32;              // 16-byte vectors of x~ per cell per batch row
};

// TMEM column map per group: D at 128 g, A buffers at 128 g + 32 + 32 b.
__device__ __forceinline__ uint32_t d_col(int g) { return 128u * g; }
__device__ __forceinline__ uint32_t a_col(int g, int b) { return 128u * g + 32u + 32u * b; }

template <int K, int CODE, int NB8>
__global__ void __launch_bounds__(kThreads, 1) gemv_tc_kernel(const TcArgs args) {
    using C = Cfg<K, CODE>;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // ---------------- shared memory carve-up
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + 960);
    uint8_t* stream = smem + 1024;
    uint8_t* bbuf = stream + kSlots * C::kUnitBytes;
    constexpr uint32_t kBlk = 256u * NB8;                              // B bytes per MMA
    constexpr uint32_t kBGroup = C::kMmaPerUnit * kBlk;
    uint8_t* zero_blk = bbuf + kGroups * kBGroup;
    uint8_t* lut = zero_blk + 256;
    const uint32_t bar0 = ptx::smem_u32(bars);
    auto full = [&](int s) { return bar0 + 8u * s; };
    auto empty = [&](int s) { return bar0 + 8u * (kSlots + s); };
    auto afull = [&](int g, int b) { return bar0 + 8u * (2 * kSlots + 2 * g + b); };
    auto aempty = [&](int g, int b) { return bar0 + 8u * (2 * kSlots + 8 + 2 * g + b); };
    auto dfull = [&](int g) { return bar0 + 8u * (2 * kSlots + 16 + g); };
    auto dempty = [&](int g) { return bar0 + 8u * (2 * kSlots + 20 + g); };

    const int64_t G = gridDim.x;
    const int64_t u0 = args.units * blockIdx.x / G, u1 = args.units * (blockIdx.x + 1) / G;
    const int nunits = (int)(u1 - u0);
    const int n_kc = (int)args.lay.n_kc;

    // ---------------- one-time setup
    {
        uint4* z = reinterpret_cast<uint4*>(bbuf);
        const int nz = (kGroups * kBGroup + 256) / 16;
        for (int i = threadIdx.x; i < nz; i += kThreads) z[i] = make_uint4(0, 0, 0, 0);
        if constexpr (C::kHyb) {
            // entry e = idx | sign << Q -> (c0, c1) with c1 negated when sign (Alg. 3), 32 replicas
            for (int i = threadIdx.x; i < (1 << (kHyBLutQ + 1)) * 8; i += kThreads) {
                const int e = i >> 3, quad = i & 7;
                uint32_t w = __ldg(args.lut + (e & ((1 << kHyBLutQ) - 1)));
                if (e >> kHyBLutQ) w ^= 0x80000000u;
                reinterpret_cast<uint4*>(lut)[(e * 128 + quad * 16) / 16] = make_uint4(w, w, w, w);
            }
        }
    }
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kSlots; ++s) {
            ptx::mbar_init(full(s), 1);
            ptx::mbar_init(empty(s), 128);
        }
        for (int g = 0; g < kGroups; ++g) {
            for (int b = 0; b < 2; ++b) {
                ptx::mbar_init(afull(g, b), 128);
                ptx::mbar_init(aempty(g, b), 1);
            }
            ptx::mbar_init(dfull(g), 1);
            ptx::mbar_init(dempty(g), 128);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(ptx::smem_u32(tmem_holder), 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_holder;

    if (warp == 0) {
        // ================= producer
        if (lane == 0) {
            for (int j = 0; j < nunits; ++j) {
                const int s = j % kSlots, use = j / kSlots;
                if (use > 0) ptx::mbar_wait(empty(s), (use - 1) & 1);
                const int64_t u = u0 + j;
                const int64_t RB = args.rb0 + u / n_kc, KC = u % n_kc;
                const uint32_t* src = args.packed + (RB * n_kc + KC) * args.lay.cell_words;
                ptx::mbar_arrive_expect_tx(full(s), C::kUnitBytes);
                ptx::bulk_g2s(ptx::smem_u32(stream + s * C::kUnitBytes), src, C::kUnitBytes, full(s));
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_f16_f32(128, kN);
            const uint32_t zaddr = ptx::smem_u32(zero_blk);
            for (int j = 0; j < nunits; ++j) {
                // unit j is the lu-th unit of group g; its handoff h is the group's (4 lu + h)-th,
                // so it uses A buffer h & 1 for the (2 lu + h/2)-th time
                const int g = j & 3;
                const uint32_t lu = (uint32_t)j >> 2;
                if (lu > 0) ptx::mbar_wait(dempty(g), (lu - 1) & 1);
                ptx::tc_fence_after();
                const uint32_t bgrp = ptx::smem_u32(bbuf + g * kBGroup);
                for (int h = 0; h < 4; ++h) {
                    const int b = h & 1;
                    ptx::mbar_wait(afull(g, b), (2 * lu + (h >> 1)) & 1);
                    ptx::tc_fence_after();
#pragma unroll
                    for (int tt = 0; tt < 2; ++tt) {
#pragma unroll
                        for (int half = 0; half < C::kMmaPerTile; ++half) {
                            const int mi = (2 * h + tt) * C::kMmaPerTile + half;
                            const uint32_t start = bgrp + mi * kBlk;
                            const uint32_t sbo = (NB8 == 2) ? 256u : (zaddr - start);
                            const uint64_t bdesc = ptx::smem_desc_kmajor_noswizzle(start, 128u, sbo);
                            const uint32_t a = tmem + a_col(g, b) + tt * C::kColsPerTile + half * 8;
                            ptx::umma_f16_ts(tmem + d_col(g), a, bdesc, idesc, (h | tt | half) != 0);
                        }
                    }
                    ptx::umma_commit(aempty(g, b));
                }
                ptx::umma_commit(dfull(g));
            }
        }
    } else {
        // ================= decoders
        const int dw = warp - 2, g = dw >> 2, q = warp & 3;
        const int tg = (dw & 3) * 32 + lane;                 // thread index within the group
        const int R = 32 * q + lane, I = R >> 4, r = R & 15;
        const uint32_t taddr_lane = tmem + ((uint32_t)(32 * q) << 16);
        const uint32_t lane4 = (uint32_t)lane * 4u;
        const uint32_t lut_base = ptx::smem_u32(lut);
        uint8_t* bgrp = bbuf + g * kBGroup;
        uint32_t lu = 0;
        for (int j = g; j < nunits; j += kGroups, ++lu) {
            const int64_t u = u0 + j;
            const int64_t RB = args.rb0 + u / n_kc, KC = u % n_kc;
            const int s = j % kSlots;
            // ---- B operand: this cell's 128 columns of x~ (rows >= B stay zero)
            for (int e = tg; e < args.B * C::kXtVecs; e += 128) {
                const int n = e / C::kXtVecs, v = e % C::kXtVecs;
                const uint4 val = *reinterpret_cast<const uint4*>(args.xt + n * args.xt_row_bytes +
                                                                  KC * (C::kXtVecs * 16) + v * 16);
                *reinterpret_cast<uint4*>(bgrp + (v >> 1) * kBlk + (n >> 3) * 256 + (v & 1) * 128 + (n & 7) * 16) = val;
            }
            ptx::fence_proxy_async_smem();
            ptx::mbar_wait(full(s), (j / kSlots) & 1);
            const uint32_t* slot = reinterpret_cast<const uint32_t*>(stream + s * C::kUnitBytes);
#pragma unroll 1
            for (int h = 0; h < 4; ++h) {
                const int b = h & 1;
                const uint32_t use = 2 * lu + (h >> 1);                // uses of A buffer b so far
                if (use > 0) ptx::mbar_wait(aempty(g, b), (use - 1) & 1);
                ptx::tc_fence_after();
                const uint32_t* pw = slot + (I * 4 + h) * (8 * K) * 2;      // word w of tile t at pw[2w + t]
                const uint32_t ta = taddr_lane + a_col(g, b);
                if constexpr (K == 2 && !C::kHyb) {
                    const uint2 A = *reinterpret_cast<const uint2*>(pw + 2 * r);
                    const uint2 Bw = *reinterpret_cast<const uint2*>(pw + 2 * ((r + 1) & 15));
#pragma unroll
                    for (int tt = 0; tt < 2; ++tt) {
                        uint32_t x[16], z[16];
                        windows_k2v1(tt ? A.y : A.x, tt ? Bw.y : Bw.x, x);
#pragma unroll
                        for (int qq = 0; qq < 16; ++qq) {
                            if constexpr (CODE == QTIP_CODE_3INST) z[qq] = inst3_word(x[qq], args.ca.a, args.ca.b, args.ca.magic);
                            else z[qq] = __dp4a(x[qq] * args.ca.a + args.ca.b, 0x01010101u, 0xE5FE6400u);
                        }
                        ptx::tmem_st16(ta + tt * 16, z);
                    }
                } else if constexpr (K == 4 && C::kHyb) {
                    const uint4 AB = *reinterpret_cast<const uint4*>(pw + 4 * r);   // words 2r, 2r+1 of both tiles
                    const uint2 Cw = *reinterpret_cast<const uint2*>(pw + 2 * ((2 * r + 2) & 31));
#pragma unroll
                    for (int tt = 0; tt < 2; ++tt) {
                        uint32_t x[8], z[8];
                        windows_k4v2_dirty(tt ? AB.y : AB.x, tt ? AB.w : AB.z, tt ? Cw.y : Cw.x, x);
#pragma unroll
                        for (int qq = 0; qq < 8; ++qq) {
                            const uint32_t h2 = x[qq] * (x[qq] + x[qq] + 2u);       // 2 (x^2 + x)
                            uint32_t off;
                            asm("lop3.b32 %0, %1, %2, %3, 0xea;" : "=r"(off) : "r"(h2), "r"(0x1FF80u), "r"(lane4));
                            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(z[qq]) : "r"(lut_base + off));
                        }
                        ptx::tmem_st8(ta + tt * 8, z);
                    }
                } else {
                    // general k (and HYB at k = 2, 3): windows from three words per tile row
                    constexpr int TW = 8 * K;
                    const int start = 16 * K * r, w0 = start >> 5, off = start & 31;
                    const uint2 W0 = *reinterpret_cast<const uint2*>(pw + 2 * (w0 % TW));
                    const uint2 W1 = *reinterpret_cast<const uint2*>(pw + 2 * ((w0 + 1) % TW));
                    const uint2 W2 = *reinterpret_cast<const uint2*>(pw + 2 * ((w0 + 2) % TW));
#pragma unroll
                    for (int tt = 0; tt < 2; ++tt) {
                        const uint32_t a0 = tt ? W0.y : W0.x, a1 = tt ? W1.y : W1.x, a2 = tt ? W2.y : W2.x;
                        if constexpr (C::kHyb) {
                            uint32_t z[8];
#pragma unroll
                            for (int qq = 0; qq < 8; ++qq) {
                                const uint32_t x = window_general(a0, a1, a2, off + qq * 2 * K);
                                const uint32_t h2 = x * (x + x + 2u);
                                uint32_t o;
                                asm("lop3.b32 %0, %1, %2, %3, 0xea;" : "=r"(o) : "r"(h2), "r"(0x1FF80u), "r"(lane4));
                                asm volatile("ld.shared.b32 %0, [%1];" : "=r"(z[qq]) : "r"(lut_base + o));
                            }
                            ptx::tmem_st8(ta + tt * 8, z);
                        } else {
                            uint32_t z[16];
#pragma unroll
                            for (int qq = 0; qq < 16; ++qq) {
                                const uint32_t x = window_general(a0, a1, a2, off + qq * K);
                                if constexpr (CODE == QTIP_CODE_3INST) z[qq] = inst3_word(x, args.ca.a, args.ca.b, args.ca.magic);
                                else z[qq] = __dp4a(x * args.ca.a + args.ca.b, 0x01010101u, 0xE5FE6400u);
                            }
                            ptx::tmem_st16(ta + tt * 16, z);
                        }
                    }
                }
                if (h == 3) ptx::mbar_arrive(empty(s));               // all reads of this slot done
                ptx::tc_wait_st();
                ptx::tc_fence_before();
                ptx::mbar_arrive(afull(g, b));
            }
            // ---- epilogue: D (row R, N columns) -> partial sums of this cell column
            ptx::mbar_wait(dfull(g), lu & 1);
            ptx::tc_fence_after();
            uint32_t d[16];
            ptx::tmem_ld16(taddr_lane + d_col(g), d);
            ptx::tc_wait_ld();
            const int64_t row = RB * kCellRows + R;
            for (int bb = 0; bb < args.B; ++bb)
                args.partial[(KC * args.B + bb) * args.lay.m_pad + row] = __uint_as_float(d[bb]) * args.code_factor;
            ptx::tc_fence_before();
            ptx::mbar_arrive(dempty(g));
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

template <int K, int CODE, int NB8>
cudaError_t launch_tc_t(const TcArgs& a, cudaStream_t s) {
    using C = Cfg<K, CODE>;
    constexpr uint32_t kBlk = 256u * NB8;
    const size_t smem = 1024 + kSlots * C::kUnitBytes + kGroups * C::kMmaPerUnit * kBlk + 256 + (C::kHyb ? kLutBytes : 0);
    auto kern = gemv_tc_kernel<K, CODE, NB8>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)std::min<int64_t>(sms, a.units);
    kern<<<grid, kThreads, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace

bool gemv_tc_supported(const Layout& lay, int code, const CodeArgs& ca, int64_t B) {
    if (B < 1 || B > 16) return false;
    if (lay.k < 2 || lay.k > 4) return false;
    if (code == QTIP_CODE_HYB && (ca.Q != kHyBLutQ || ca.two_sign)) return false;
    return true;
}

int gemv_tc_xt_mode(int code) { return code == QTIP_CODE_HYB ? 2 : 1; }

cudaError_t launch_gemv_tc(const Layout& lay, int code, const CodeArgs& ca, const void* packed, const uint16_t* lut,
                           const void* xt_compact, int64_t xt_row_bytes, int64_t B, int64_t rb0, int64_t rb1,
                           float* partial, cudaStream_t s) {
    TcArgs a;
    a.packed = (const uint32_t*)packed;
    a.lay = lay;
    a.ca = ca;
    a.lut = (const uint32_t*)lut;
    a.xt = (const uint8_t*)xt_compact;
    a.xt_row_bytes = xt_row_bytes;
    a.B = (int)B;
    a.rb0 = rb0;
    a.units = (rb1 - rb0) * lay.n_kc;
    a.code_factor = (code == QTIP_CODE_1MAD) ? 5.0f / 739.0f : 1.0f;   // 1/147.8 for 1MAD
    a.partial = partial;
    const bool nb2 = B > 8;
    cudaError_t e = cudaErrorInvalidValue;
#define QTIP_TC_CASE(KK, CC)                                                         \
    if (lay.k == KK && code == CC) e = nb2 ? launch_tc_t<KK, CC, 2>(a, s) : launch_tc_t<KK, CC, 1>(a, s);
    QTIP_TC_CASE(2, QTIP_CODE_3INST)
    QTIP_TC_CASE(3, QTIP_CODE_3INST)
    QTIP_TC_CASE(4, QTIP_CODE_3INST)
    QTIP_TC_CASE(2, QTIP_CODE_1MAD)
    QTIP_TC_CASE(3, QTIP_CODE_1MAD)
    QTIP_TC_CASE(4, QTIP_CODE_1MAD)
    QTIP_TC_CASE(2, QTIP_CODE_HYB)
    QTIP_TC_CASE(3, QTIP_CODE_HYB)
    QTIP_TC_CASE(4, QTIP_CODE_HYB)
#undef QTIP_TC_CASE
    count_launch(1);
    return e;
}

}  // namespace qtip
