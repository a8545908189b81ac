// k_gemv_row.cu -- row-tile fused trellis-decode GEMV (impl 4), the batch <= 4 latency path.
//
// One CTA per tile row (16 output rows).  Its W warps split the row's cells (128-column blocks of
// the packed layout; warp w takes cells w, w + W, ...), each decoding the 8 tiles of its cells
// straight into mma.sync A fragments (mma_tile.cuh) and accumulating in registers.  The warps'
// sums are added in warp order through shared memory and the CTA writes finished y~ rows:
// no split-K partials in global memory, no reduction kernel, and each row's arithmetic depends
// only on n (deterministic, and a row shard reproduces the full call bit for bit).
//
// Each warp streams its cells through a private ring of cp.async.bulk stages (the cell's tile-row
// chunk of the packed stream, 256 k bytes, plus the cell's x~ columns), refilled by its lane 0:
// no CTA-wide barrier until the final sum.  The packed weights do not depend on the previous
// kernel, so the first stages are requested before the PDL wait and stream in while the RHT-in
// still runs; only the x~ copies wait for it.
#include <algorithm>

#include "internal.h"
#include "mma_tile.cuh"
#include "tc.cuh"
#include "trace.cuh"

namespace qtip {
namespace {

using namespace mma;

constexpr int kRowMaxWarps = 16;
constexpr int kRowMaxStages = 4;

__device__ unsigned long long* g_row_trace = nullptr;
__device__ int g_row_trace_cap = 0;

struct RowArgs {
    const uint32_t* packed;
    Layout lay;
    CodeArgs ca;
    const uint32_t* lut;       // HYB: 2^Q words (c0 | c1 << 16)
    const uint32_t* xt;        // fragment-ordered x~ rows of xt_row_words u32
    int64_t xt_row_words;
    int B;
    int stages;                // per-warp ring depth
    int64_t tile_row0;         // first tile row of this launch
    float code_factor;
    float* y;                  // y[b * y_stride + (i - row_lo)] for rows i in [row_lo, row_hi)
    int64_t y_stride;
    int64_t row_lo, row_hi;
    float scale;
};

// W = blockDim.x / 32 warps per tile row (16, 8 or 4: the launcher picks the widest that keeps
// every CTA resident in one wave); registers are capped at 64 so two 16-warp CTAs fit an SM.
template <int K, int CODE, bool kImm>
__global__ void __launch_bounds__(32 * kRowMaxWarps, 2) gemv_row_kernel(const RowArgs args) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr bool kHyb = CODE == QTIP_CODE_HYB;
    constexpr int TW = 8 * K;
    constexpr uint32_t kChunkBytes = 256u * K;                       // one cell's 8 tiles of this tile row
    constexpr uint32_t kXRowBytes = kHyb ? 256u : 512u;              // x~ of one cell, one batch row
    const int S = args.stages;
    // x~ rows padded by 64 B (3INST/1MAD) / 32 B (HYB) when B > 1: the batch rows of a B-fragment
    // load then spread over all bank groups (unpadded: up to 8-way conflicts at B = 8)
    const uint32_t xstride = args.B > 1 ? (kHyb ? 288u : 576u) : kXRowBytes;
    const uint32_t stage_bytes = kChunkBytes + xstride * (uint32_t)args.B;   // rows >= B are not staged
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int W = blockDim.x >> 5;
    const int g = lane >> 2, tig = lane & 3;
    const int64_t n_kc = args.lay.n_kc;
    const int64_t I = args.tile_row0 + blockIdx.x;                  // tile row
    const int64_t RB = I / kCellTileRows, Il = I % kCellTileRows;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem) + warp * kRowMaxStages;
    float* red = reinterpret_cast<float*>(smem + 8 * kRowMaxWarps * kRowMaxStages);   // [W][16][B]
    uint8_t* ring = smem + 8 * kRowMaxWarps * kRowMaxStages + 4 * kRowMaxWarps * kTile * args.B;
    ring += (size_t)warp * S * stage_bytes;
    const CodeArgs ca = args.ca;
    const Lcg<CODE, kImm> lcg(ca);
    const int ncells = (int)((n_kc - warp + W - 1) / W);                   // cells warp, warp + W, ...
    __shared__ unsigned long long trace_ts[4];
    CtaTrace trace{trace_ts};
    trace.entry(g_row_trace);

    if (lane == 0) {
        for (int st = 0; st < S; ++st) ptx::mbar_init(ptx::smem_u32(full + st), 1);
        ptx::fence_mbar_init();
    }
    __syncwarp();
    auto issue_w = [&](int j) {                                      // lane 0: packed chunk of cell j
        const int st = j % S;
        const int64_t kc = warp + (int64_t)j * W;
        const uint32_t bar = ptx::smem_u32(full + st);
        ptx::mbar_arrive_expect_tx(bar, kChunkBytes + kXRowBytes * (uint32_t)args.B);   // bytes copied (not the padded stage)
        ptx::bulk_g2s_stream(ptx::smem_u32(ring + st * stage_bytes),
                      args.packed + (RB * n_kc + kc) * (int64_t)(512 * K) + Il * (kChunkBytes / 4), kChunkBytes, bar);
    };
    auto issue_x = [&](int j) {                                      // lane 0: x~ columns of cell j
        const int st = j % S;
        const int64_t kc = warp + (int64_t)j * W;
        for (int n = 0; n < args.B; ++n)
            ptx::bulk_g2s(ptx::smem_u32(ring + st * stage_bytes + kChunkBytes + n * xstride),
                          reinterpret_cast<const uint8_t*>(args.xt) + n * args.xt_row_words * 4 + kc * kXRowBytes,
                          kXRowBytes, ptx::smem_u32(full + st));
    };
    if (lane == 0)
        for (int j = 0; j < min(ncells, S); ++j) issue_w(j);
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    trace.waited(g_row_trace);
    if (lane == 0)
        for (int j = 0; j < min(ncells, S); ++j) issue_x(j);

    float acc[1][4] = {{0.0f, 0.0f, 0.0f, 0.0f}};
    for (int j = 0; j < ncells; ++j) {
        const int st = j % S;
        ptx::mbar_wait_sleep(ptx::smem_u32(full + st), (j / S) & 1);
        const uint32_t* chunk = reinterpret_cast<const uint32_t*>(ring + st * stage_bytes);
        const uint32_t* xs = reinterpret_cast<const uint32_t*>(ring + st * stage_bytes + kChunkBytes);
#pragma unroll
        for (int pp = 0; pp < kCellTileCols / 2; ++pp) {
            uint32_t bf[2][1][4];
            load_bfrag<1, kHyb>(xs, (int)(xstride / 4), 2 * pp, g, tig, args.B, bf[0]);
            load_bfrag<1, kHyb>(xs, (int)(xstride / 4), 2 * pp + 1, g, tig, args.B, bf[1]);
            tile_pair<K, CODE, 1, kImm>(chunk + pp * TW * 2, bf, acc, g, tig, lcg, ca, args.lut);
        }
        __syncwarp();                                                // every lane is done with stage st
        if (lane == 0 && j + S < ncells) {
            issue_w(j + S);
            issue_x(j + S);
        }
    }
    // acc[0][e] = D[MMA row g + 8 (e >> 1)][batch 2 tig + (e & 1)]; MMA row g <-> tile row 2g,
    // g + 8 <-> 2g + 1
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int b = 2 * tig + (e & 1), r = 2 * g + (e >> 1);
        if (b < args.B) red[(warp * kTile + r) * args.B + b] = acc[0][e];
    }
    __syncthreads();
    trace.aux(g_row_trace, 1);
    for (int t = threadIdx.x; t < kTile * args.B; t += blockDim.x) {
        const int r = t % kTile, b = t / kTile;
        const int64_t i = I * kTile + r;
        if (i < args.row_lo || i >= args.row_hi) continue;
        float s = 0.0f;
        for (int w = 0; w < W; ++w) s += red[(w * kTile + r) * args.B + b];
        args.y[b * args.y_stride + (i - args.row_lo)] = args.scale * (s * args.code_factor);
    }
    trace.exit(g_row_trace, 4, g_row_trace_cap);
}

template <int K, int CODE, bool kImm>
cudaError_t launch_row_t(RowArgs a, int64_t tile_rows, cudaStream_t s) {
    constexpr bool kHyb = CODE == QTIP_CODE_HYB;
    auto kern = gemv_row_kernel<K, CODE, kImm>;
    const size_t stage = 256u * K + (a.B > 1 ? (kHyb ? 288u : 576u) : (kHyb ? 256u : 512u)) * (size_t)a.B;
    const size_t fixed = 8 * kRowMaxWarps * kRowMaxStages + 4 * kRowMaxWarps * kTile * (size_t)a.B;
    // widest W whose CTAs all fit in one wave (per-SM CTA count from registers / threads, and a
    // shared-memory share of 227 KB / CTAs); ring depth as deep as that share allows (2..4)
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    const int regs = fa.numRegs > 0 ? fa.numRegs : 64;
    int W = 4, per_sm = 1;
    for (int w : {16, 8, 4}) {
        per_sm = std::min(65536 / (regs * 32 * w), 2048 / (32 * w));
        W = w;
        if ((int64_t)per_sm * num_sms() >= tile_rows) break;
    }
    const size_t share = std::min<size_t>(227 * 1024 / std::max(per_sm, 1), 200 * 1024);
    int S = (int)((share - fixed) / (W * stage));
    S = S < 2 ? 2 : (S > kRowMaxStages ? kRowMaxStages : S);
    a.stages = S;
    const size_t smem = fixed + (size_t)W * S * stage;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, dim3((unsigned)tile_rows), dim3(32 * W), smem, s, a);
}

}  // namespace

cudaError_t set_cta_trace_row(unsigned long long* buf, int cap) {
    cudaError_t e = cudaMemcpyToSymbol(g_row_trace, &buf, sizeof(buf));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_row_trace_cap, &cap, sizeof(cap));
    return e;
}

bool gemv_row_supported(const Layout& lay, int code, const CodeArgs& ca, int64_t B) {
    if (B < 1 || B > 4) return false;
    if (lay.k < 2 || lay.k > 4) return false;
    if (code == QTIP_CODE_HYB && ca.two_sign) return false;
    return true;
}

cudaError_t launch_gemv_row(const Layout& lay, int code, const CodeArgs& ca, const void* packed, const uint16_t* lut,
                            const void* xt_frag, int64_t xt_row_words, int64_t B, int64_t row_begin, int64_t row_end,
                            float* y, int64_t y_stride, int64_t row_lo, int64_t row_hi, float scale, cudaStream_t s) {
    RowArgs a;
    a.packed = (const uint32_t*)packed;
    a.lay = lay;
    a.ca = ca;
    a.lut = (const uint32_t*)lut;
    a.xt = (const uint32_t*)xt_frag;
    a.xt_row_words = xt_row_words;
    a.B = (int)B;
    a.tile_row0 = row_begin / kTile;
    a.code_factor = (code == QTIP_CODE_1MAD) ? 5.0f / 739.0f : 1.0f;
    a.y = y;
    a.y_stride = y_stride;
    a.row_lo = row_lo;
    a.row_hi = row_hi;
    a.scale = scale;
    const int64_t tile_rows = (row_end + kTile - 1) / kTile - a.tile_row0;
    const bool imm = code != QTIP_CODE_HYB && ca.a == (code == QTIP_CODE_1MAD ? 34038481u : 89226354u) &&
                     ca.b == (code == QTIP_CODE_1MAD ? 76625530u : 64248484u);
    cudaError_t e = cudaErrorInvalidValue;
#define QTIP_ROW_CASE(KK, CC)                                                          \
    if (lay.k == KK && code == CC) e = imm ? launch_row_t<KK, CC, true>(a, tile_rows, s) \
                                           : launch_row_t<KK, CC, false>(a, tile_rows, s);
    QTIP_ROW_CASE(2, QTIP_CODE_3INST)
    QTIP_ROW_CASE(3, QTIP_CODE_3INST)
    QTIP_ROW_CASE(4, QTIP_CODE_3INST)
    QTIP_ROW_CASE(2, QTIP_CODE_1MAD)
    QTIP_ROW_CASE(3, QTIP_CODE_1MAD)
    QTIP_ROW_CASE(4, QTIP_CODE_1MAD)
    QTIP_ROW_CASE(2, QTIP_CODE_HYB)
    QTIP_ROW_CASE(3, QTIP_CODE_HYB)
    QTIP_ROW_CASE(4, QTIP_CODE_HYB)
#undef QTIP_ROW_CASE
    count_launch(1);
    return e;
}

}  // namespace qtip
