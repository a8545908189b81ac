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
#include "internal.h"
#include "mma_tile.cuh"
#include "tc.cuh"
#include "trace.cuh"

namespace qtip {
namespace {

constexpr int kMmaWarps = 4;

__device__ unsigned long long* g_mma_trace = nullptr;
__device__ int g_mma_trace_cap = 0;
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
    MmaEpilogue ep;
};

using namespace mma;

// Fused split-K reduction of row block RB by the last CTA to finish one of its cells: rows
// i of the block, y[b][i - row_lo] = scale * sum_kc partial[kc][b][i] with launch_reduce's
// association (eight interleaved kc slices summed in increasing kc, then added in slice order).
__device__ __forceinline__ void reduce_row_block(const MmaArgs& args, int64_t RB) {
    const int64_t n_kc = args.lay.n_kc, m_pad = args.lay.m_pad;
    for (int t = threadIdx.x; t < kCellRows * args.B; t += blockDim.x) {
        const int b = t / kCellRows;
        const int64_t i = RB * kCellRows + (t % kCellRows);
        if (i < args.ep.row_lo || i >= args.ep.row_hi) continue;
        const float* p = args.partial + (int64_t)b * m_pad + i;
        const int64_t step = (int64_t)args.B * m_pad;
        float sl[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        int64_t kc = 0;
        for (; kc < n_kc; kc += 32) {                               // 32 loads in flight per thread
            float v[32];                                            // (+0 past n_kc: sums unchanged)
#pragma unroll
            for (int q = 0; q < 32; ++q) v[q] = kc + q < n_kc ? __ldcg(p + (kc + q) * step) : 0.0f;
#pragma unroll
            for (int q = 0; q < 32; ++q) sl[q & 7] += v[q];
        }
        float tot = 0.0f;
#pragma unroll
        for (int q = 0; q < 8; ++q) tot += sl[q];
        args.ep.y[b * args.ep.y_stride + (i - args.ep.row_lo)] = args.ep.scale * tot;
    }
}

template <int K, int CODE, int NG, bool kImm>   // NG = batch groups of 8 (1 or 2); kImm = paper LCG constants
__global__ void __launch_bounds__(32 * kMmaWarps, (K == 2 && NG == 1) ? 8 : (NG == 2 ? 4 : 6)) gemv_mma_kernel(const MmaArgs args) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr bool kHyb = CODE == QTIP_CODE_HYB;
    constexpr int TW = 8 * K;
    constexpr uint32_t kCellBytes = 2048u * K;                      // packed stream of one cell
    constexpr uint32_t kXRowBytes = kHyb ? 256u : 512u;              // x~ of one cell, one batch row
    // x~ rows padded by 64 B (3INST/1MAD) / 32 B (HYB) when B > 1: the batch rows of a B-fragment
    // load then spread over all bank groups (unpadded: up to 8-way conflicts at B = 8)
    const uint32_t xstride = args.B > 1 ? (kHyb ? 288u : 576u) : kXRowBytes;
    const uint32_t stage_bytes = kCellBytes + xstride * (uint32_t)args.B;   // rows >= B are not staged
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);             // kMmaStages mbarriers
    __shared__ int s_last;
    uint8_t* stages = smem + 128;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, tig = lane & 3;
    const int n_kc = (int)args.lay.n_kc;
    const int64_t G = gridDim.x;
    const CodeArgs ca = args.ca;
    const Lcg<CODE, kImm> lcg(ca);
    __shared__ unsigned long long trace_ts[4];
    __shared__ int64_t s_unit[kMmaStages];                           // cell of each ring stage (-1: done)
    CtaTrace trace{trace_ts};
    trace.entry(g_mma_trace);

    if (threadIdx.x == 0) {
        for (int st = 0; st < kMmaStages; ++st) ptx::mbar_init(ptx::smem_u32(full + st), 1);
        ptx::fence_mbar_init();
    }
    __syncthreads();
    // Work distribution: ring round r < kMmaStages of CTA c takes cell c + r G (static, so its
    // weights can be requested before the PDL wait); later cells come from a global counter
    // (zeroed by the input kernel) in increasing order, so row blocks complete in order and the
    // split-K tail is one cell, not one CTA's share.
    auto issue_x = [&](int st, int64_t u) {                          // thread 0: x~ columns of cell u
        const int64_t KC = u % n_kc;
        uint8_t* dst = stages + st * stage_bytes + kCellBytes;
        for (int n = 0; n < args.B; ++n)
            ptx::bulk_g2s(ptx::smem_u32(dst + n * xstride),
                          reinterpret_cast<const uint8_t*>(args.xt) + n * args.xt_row_words * 4 + KC * kXRowBytes,
                          kXRowBytes, ptx::smem_u32(full + st));
    };
    auto issue_w = [&](int st, int64_t u) {                          // thread 0: packed stream of cell u
        const uint32_t bar = ptx::smem_u32(full + st);
        const int64_t RB = args.rb0 + u / n_kc, KC = u % n_kc;
        ptx::mbar_arrive_expect_tx(bar, kCellBytes + kXRowBytes * (uint32_t)args.B);
        ptx::bulk_g2s_stream(ptx::smem_u32(stages + st * stage_bytes),
                      args.packed + (RB * n_kc + KC) * (int64_t)(kCellBytes / 4), kCellBytes, bar);
    };
    // the packed weights never depend on the previous kernel: start streaming them before the
    // PDL wait (overlapping the RHT-in); x~, the counters and the workspace only after it
    if (threadIdx.x == 0)
        for (int st = 0; st < kMmaStages; ++st) {
            const int64_t u = blockIdx.x + st * G;
            s_unit[st] = u < args.units ? u : -1;
            if (u < args.units) issue_w(st, u);
        }
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    trace.waited(g_mma_trace);
    int pending = 0;                                                 // thread 0: next counter ticket
    if (threadIdx.x == 0) {
        for (int st = 0; st < kMmaStages; ++st) {
            const int64_t u = s_unit[st];
            if (u >= 0) issue_x(st, u);
            else ptx::mbar_arrive(ptx::smem_u32(full + st));         // "done" marker, no data
        }
        pending = atomicAdd(args.ep.cnt + args.ep.n_rb, 1);          // ticket for the next free stage
    }

    int j = 0;
    for (;; ++j) {
        const int st = j % kMmaStages;
        ptx::mbar_wait_sleep(ptx::smem_u32(full + st), (j / kMmaStages) & 1);
        const int64_t u = s_unit[st];
        if (u < 0) break;
        const int64_t RB = args.rb0 + u / n_kc, KC = u % n_kc;
        const uint32_t* cell = reinterpret_cast<const uint32_t*>(stages + st * stage_bytes);
        const uint32_t* xs = reinterpret_cast<const uint32_t*>(stages + st * stage_bytes + kCellBytes);
        float acc[2][NG][4];
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int ng = 0; ng < NG; ++ng) acc[t][ng][0] = acc[t][ng][1] = acc[t][ng][2] = acc[t][ng][3] = 0.0f;
#pragma unroll
        for (int pp = 0; pp < kCellTileCols / 2; ++pp) {              // tile pair (2pp, 2pp+1)
            uint32_t bf[2][NG][4];                                   // shared by the warp's two tile rows
            load_bfrag<NG, kHyb>(xs, (int)(xstride / 4), 2 * pp, g, tig, args.B, bf[0]);
            load_bfrag<NG, kHyb>(xs, (int)(xstride / 4), 2 * pp + 1, g, tig, args.B, bf[1]);
#pragma unroll
            for (int tr = 0; tr < 2; ++tr) {
                const int I = 2 * warp + tr;
                tile_pair<K, CODE, NG, kImm>(cell + (I * 4 + pp) * TW * 2, bf, acc[tr], g, tig, lcg, ca, args.lut);
            }
        }
        __syncthreads();                                             // every warp is done with stage st
        if (threadIdx.x == 0) {                                      // refill stage st (or mark done)
            const int64_t un = s_unit[st] < 0 ? -1 : (int64_t)kMmaStages * G + pending;
            if (un >= 0 && un < args.units) {
                s_unit[st] = un;
                issue_w(st, un);
                issue_x(st, un);
                pending = atomicAdd(args.ep.cnt + args.ep.n_rb, 1);  // its latency hides behind a cell
            } else {
                s_unit[st] = -1;
                ptx::mbar_arrive(ptx::smem_u32(full + st));
            }
        }
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
        // ---- last CTA to finish a cell of row block RB reduces the block: the CTA barrier orders
        //      every thread's partial stores before thread 0's (cumulative) gpu-scope release
        if (args.ep.y == nullptr) continue;                          // split-K reduced by launch_reduce
        __syncthreads();
        if (threadIdx.x == 0) {
            int old;
            asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;" : "=r"(old) : "l"(args.ep.cnt + RB) : "memory");
            s_last = old == n_kc - 1;
        }
        __syncthreads();
        if (s_last) {                                                // acquire by thread 0, barrier-propagated
            trace.aux(g_mma_trace, (unsigned long long)RB + 1);
            reduce_row_block(args, RB);
            if (threadIdx.x == 0) args.ep.cnt[RB] = 0;                // left zero for the next call
        }
    }
    // the last CTA to leave resets the work counter and the exit counter: every launch (and the
    // next one, which reads them only after its PDL wait) starts from zero
    if (threadIdx.x == 0) {
        int* work = args.ep.cnt + args.ep.n_rb;
        int old;
        asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;" : "=r"(old) : "l"(work + 1) : "memory");
        if (old == (int)G - 1) {
            work[0] = 0;
            work[1] = 0;
        }
    }
    trace.exit(g_mma_trace, 3 | (j << 8), g_mma_trace_cap);
}

template <int K, int CODE, int NG, bool kImm>
cudaError_t launch_mma_t(const MmaArgs& a, cudaStream_t s) {
    constexpr bool kHyb = CODE == QTIP_CODE_HYB;
    const size_t xstride = a.B > 1 ? (kHyb ? 288u : 576u) : (kHyb ? 256u : 512u);   // as in the kernel
    const size_t smem = 128 + (size_t)kMmaStages * (2048u * K + xstride * (size_t)a.B);
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

cudaError_t set_cta_trace_mma(unsigned long long* buf, int cap) {
    cudaError_t e = cudaMemcpyToSymbol(g_mma_trace, &buf, sizeof(buf));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_mma_trace_cap, &cap, sizeof(cap));
    return e;
}

int gemv_mma_xt_mode(int code) { return code == QTIP_CODE_HYB ? 4 : 3; }
int gemv_mma_batch_pad(int64_t B) { return B > 8 ? 16 : 8; }

cudaError_t launch_gemv_mma(const Layout& lay, int code, const CodeArgs& ca, const void* packed, const uint16_t* lut,
                            const void* xt_frag, int64_t xt_row_words, int64_t B, int64_t rb0, int64_t rb1,
                            float* partial, const MmaEpilogue& ep, cudaStream_t s) {
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
    a.ep = ep;
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
