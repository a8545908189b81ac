// k_umma.cu -- impl 7: stream-K fused trellis-decode GEMV/GEMM on the 5th-generation tensor cores.
//
//   y~[rows] = W~[rows, :] x~        (PAPER.md:96-97 inner product; W~ tiles P:389-390, codes Alg. 1-3)
//
// Work = the launch's 128 x 128 cells (8 x 8 tiles of T = 256), of G same-shape
// layers stacked into one "virtual" matrix (grouped q,k,v / gate,up launches).  The U cells are cut
// into W = P equal contiguous ranges in row-major order (stream-K): range w is
// [U w / W, U (w+1) / W), CTA i runs range i.  Every CTA gets the same number of cells
// (+-1), whatever the shape: no tile-row imbalance and no one-wave rule.
//
// One CTA per SM, 18 warps:
//   warp 0      producer: one TMA stream of (x~ slab, weight cell) pairs.  Weight cells (2048k bytes,
//               L2 evict-first) go into an S-stage ring; the first S are requested before the PDL
//               wait (the weights do not depend on the previous kernel), so the ring fills while it
//               finishes.  After the wait, the x~ slab of each cell's column (128 columns x BP batch
//               rows, binary16) goes into an XS-slot ring just ahead of the cell's weights; a slot is
//               refilled once the MMAs that read it completed.  The slab ring replaces a whole-range
//               x~ window: any batch width fits shared memory in one pass, so no pass boundary drains
//               the pipeline (HYB B = 16: 3 passes before).
//   warp 1      MMA issuer (one elected thread): for every cell, waits for its decoded A operand in
//               TMEM and issues 8 tcgen05.mma (kind::f16, M = 128, N = 16/64, K = 16, A from TMEM,
//               B = x~ from shared memory, D in TMEM) -- asynchronous, so the tensor core never
//               stalls the integer decode (the register-fed mma.sync of impls 3-6 serialises with
//               it: DESIGN 5.1).  The D accumulator of a row block ("segment") lives in TMEM across
//               the range (double-buffered between segments); tcgen05.commit hands it to the epilogue.
//               Measured (scripts/umma_rate.cu): an M=128, K=16 MMA costs ~56 cycles for any N <= 64,
//               so a cell (8 MMAs) takes ~450 cycles: 36 weights/clk/SM, above the decode rate.
//   warps 2-5   epilogue (the four TMEM lane quadrants): tcgen05.ld of the finished D (thread = row), scale, store the segment's partial sums (128 rows x B).
//   warps 6-17  three decoder groups of four warps (one warp per TMEM lane quadrant); cell j goes to
//               group j mod 3.  Thread = one row of the cell (TMEM lane): it reads its row's stream
//               words of a tile pair from the ring (LDS.64/128), extracts the 16 trellis windows of
//               each tile row, evaluates the code and writes the A operand of its
//               row straight into its TMEM lane with tcgen05.st (32x32b): binary16 weights, two per
//               32-bit column.  3INST (Alg. 2): m1 + m2 summed in binary16 (HADD2, the paper's
//               footnote P:265 -- exactly qtip_decode's value); 1MAD (Alg. 1): the exact integer
//               s - 510 as binary16 (dp4a half2(1024 + s, -1534) summed), 1/147.8 applied to the
//               sums; HYB (Alg. 3): a sign-folded, 32-way replicated shared-memory LUT.  Two TMEM A
//               buffers per group (a whole cell each), hand-off through mbarriers.
//
// Partial sums: a row block that lies in one range is written straight to y~ by the epilogue.  A row
// block split between ranges gets one segment (128 rows x B partial sums) per range, and the last of
// those ranges to arrive (an atomic ticket per row block, zero between launches) adds them in range
// order -- a fixed association, so the result is deterministic for a given (shape, row range, batch,
// SM count).  Segment ids are w - w_first(layer) + row block (injective because ranges are ordered).
//
// x~ in shared memory, the UMMA B operand (K-major, SWIZZLE_NONE): element k of batch row r at byte
// (k / 8) * 16 BP + 16 r + 2 (k % 8) of its cell column's slab, BP = batch padded to a power of two.
// The descriptor's leading byte offset (K direction) is 16 BP: for BP < 8 the core matrices' rows
// >= BP overlap the next K chunks (or, for the last chunk of a slab, the next slot / the ring's
// padding) -- they only feed accumulator columns >= B, which are never read -- so a slab costs
// exactly 256 BP bytes.
#include <algorithm>

#include "internal.h"
#include "umma_decode.cuh"

namespace qtip {
namespace {

constexpr int kUG = 3;                       // decoder groups
constexpr int kUWarps = 6 + 4 * kUG;
constexpr int kUThreads = 32 * kUWarps;      // 576
constexpr int kMaxXS = 32;                   // x~ slab slots (at most)
constexpr uint32_t kLutQ = 9;
constexpr uint32_t kLutBytes = (1u << (kLutQ + 1)) * 128u;   // 1024 sign-folded entries x 32 replicas x 4 B
constexpr uint32_t kHdr = 1024;              // barriers, TMEM base
constexpr int kNBuf = 2;                     // A buffers (one cell each) per decoder group

// ring stages per (k, code): the HYB LUT takes 128 KB of shared memory
__host__ __device__ constexpr int umma_stages(int K, int code) { return code == QTIP_CODE_HYB ? 6 : (K == 2 ? 12 : 8); }

struct UmmaArgs {
    const uint32_t* packed[kMaxGroup];
    const uint8_t* xt[kMaxGroup];            // x~ (B layout above), all n_kc columns
    float* seg[kMaxGroup];                   // [(W + nrb)][BP][128] fp32 per layer
    int* ticket[kMaxGroup];                  // [nrb] arrival counters per layer (zero between launches)
    float* yout[kMaxGroup];                  // y~ (or scale * y~) rows [0, rows) of the launch, batch stride ys
    float yscale[kMaxGroup];                 // scale of the written rows (includes 1MAD's 1/147.8)
    int64_t ys, rows;
    const uint32_t* lut;                     // HYB: 2^Q words (c0 | c1 << 16), shared by the group
    Layout lay;
    CodeArgs ca;
    int G;
    int64_t rb0;                             // row blocks [rb0, rb0 + nrb) of every layer
    int nrb;
    int U;                                   // cells = G * nrb * n_kc (U * W < 2^32: 32-bit index math)
    int W;                                   // ranges
    int B, BP;
    float code_factor;
    uint32_t off_ring, off_x, off_rec;       // shared-memory offsets (LUT at kHdr; MMA cell records)
    uint32_t xcol_bytes;                     // x~ bytes per cell column (one slab)
    int XS;                                  // x~ slab slots
    uint32_t lbo, sbo;
};

// Debug timeline of CTA 0 (qtip_internal_set_umma_trace; null in normal operation): u64 clock64
// stamps at [kind * 64 + index].  The pointer is read once per thread at kernel start.
__device__ unsigned long long* g_umma_trace = nullptr;
__device__ int g_umma_trace_cta = 0;                 // the traced CTA
__device__ __forceinline__ void utrace_at(unsigned long long* t, int kind, int64_t idx) {
    if (t != nullptr && idx < 64) t[kind * 64 + idx] = clock64();
}
#define utrace(kind, idx) utrace_at(trc, (kind), (idx))

__device__ __forceinline__ int range_lo(int U, int W, int w) { return (int)((uint32_t)U * (uint32_t)w / (uint32_t)W); }
// range containing cell u: the largest w with U w / W <= u
__device__ __forceinline__ int range_of(int U, int W, int u) {
    return (int)((((uint32_t)u + 1u) * (uint32_t)W - 1u) / (uint32_t)U);
}

__device__ __forceinline__ void warp_arrive(uint32_t bar, int lane) {
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(bar);
}

// ---------------------------------------------------------------------------------------- kernel
template <int K, int CODE, int N, bool kImm>
__global__ void __launch_bounds__(kUThreads, 1) umma_gemv_kernel(const __grid_constant__ UmmaArgs a) {
    constexpr bool kHyb = CODE == QTIP_CODE_HYB;
    constexpr int S = umma_stages(K, CODE);
    constexpr uint32_t kCellBytes = 2048u * K;
    constexpr int kTW = 8 * K;
    constexpr uint32_t kACols = 64;                          // one cell: 128 binary16 weights per row
    constexpr uint32_t kD1 = N;                              // second D buffer
    constexpr uint32_t kA0 = 2 * N <= 128 ? 128u : 2 * N;
    static_assert(kA0 + kUG * kNBuf * kACols <= 512, "TMEM budget");
    constexpr uint32_t idesc = ptx::idesc_f16_f32(128, N);

    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    unsigned long long* const trc = (int)blockIdx.x == g_umma_trace_cta ? g_umma_trace : nullptr;
    const uint32_t bar0 = ptx::smem_u32(smem);
    auto full = [&](int s) { return bar0 + 8u * s; };
    auto empty = [&](int s) { return bar0 + 8u * (S + s); };
    auto afull = [&](int g, int b) { return bar0 + 8u * (2 * S + g * kNBuf + b); };
    auto aempty = [&](int g, int b) { return bar0 + 8u * (2 * S + kUG * kNBuf + g * kNBuf + b); };
    const uint32_t barD = bar0 + 8u * (2 * S + 2 * kUG * kNBuf);
    auto dfull = [&](int d) { return barD + 8u * d; };
    auto dempty = [&](int d) { return barD + 16u + 8u * d; };
    auto xfull = [&](int x) { return barD + 32u + 8u * x; };
    auto xempty = [&](int x) { return barD + 32u + 8u * (kMaxXS + x); };
    const int XS = a.XS;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + 1016);
    uint8_t* ring = smem + a.off_ring;
    const uint32_t xwin = ptx::smem_u32(smem + a.off_x);
    const int n_kc = (int)a.lay.n_kc;
    const int Ul = a.nrb * n_kc;                              // cells per layer
    const int P = (int)gridDim.x;

    // ---------------- setup (static data only: overlaps the previous kernel under PDL)
    if constexpr (kHyb) {
        // entry e = idx | sign << 9 -> (c0, c1) with c1 negated for sign (Alg. 3), replica r at
        // word 32 e + r: conflict-free LDS for any entries.  512 threads x 16 consecutive-lane vector
        // stores, all 16 loads issued first (one dependent L2 load per store was ~10 % of a launch:
        // ncu, profiles/r2s3)
        uint4* lt = reinterpret_cast<uint4*>(smem + kHdr);
        constexpr int kFill = (1 << (kLutQ + 1)) * 8 / 512;  // 16
        if (threadIdx.x < 512) {
            uint32_t w[kFill];
#pragma unroll
            for (int k = 0; k < kFill; ++k) {
                const int e = (threadIdx.x + 512 * k) >> 3;
                w[k] = __ldg(a.lut + (e & ((1 << kLutQ) - 1))) ^ ((e >> kLutQ) ? 0x80000000u : 0u);
            }
#pragma unroll
            for (int k = 0; k < kFill; ++k) lt[threadIdx.x + 512 * k] = make_uint4(w[k], w[k], w[k], w[k]);
        }
    }
    if (warp == 0) {
        if (lane == 0) {
            for (int s = 0; s < S; ++s) {
                ptx::mbar_init(full(s), 1);
                ptx::mbar_init(empty(s), 4);                  // the decoding group's four warps
            }
            for (int g = 0; g < kUG; ++g)
                for (int b = 0; b < kNBuf; ++b) {
                    ptx::mbar_init(afull(g, b), 4);
                    ptx::mbar_init(aempty(g, b), 1);
                }
            for (int d = 0; d < 2; ++d) {
                ptx::mbar_init(dfull(d), 1);
                ptx::mbar_init(dempty(d), 4);
            }
            for (int x = 0; x < XS; ++x) {
                ptx::mbar_init(xfull(x), 1);
                ptx::mbar_init(xempty(x), 1);
            }
            ptx::fence_mbar_init();
        }
        __syncwarp();
        ptx::tmem_alloc(ptx::smem_u32(tmem_holder), 512);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_holder, 0);
    if (threadIdx.x == 0) ptx::pdl_launch_dependents();
    if (threadIdx.x == 0) utrace(7, 0);

    // Every role loop is warp-uniform (values in uniform registers; one elected lane issues copies and
    // MMAs) and advances its counters incrementally: a 64-bit division or lane-0-only code per cell
    // costs hundreds of cycles.
    if (warp == 0) {
        // ================= producer: one TMA stream of (x~ slab, weight cell) pairs in the CTA's cell
        // order.  The weights do not depend on the previous kernel: the first S cells are requested
        // before the PDL wait; the x~ slabs (the previous kernel's output) after it, each one ahead of
        // its cell's weights, so a slab never waits behind later weight cells in the SM's TMA queue
        // (a separate x~ warp's copies did: traced MMA cadence 700 -> 1000 cycles per cell).
        // Its per-cell path is kept short (incremental cursors, one elected issue block): the warp
        // shares its sub-partition with three decoder warps (traced: ~350 cycles per bulk-copy issue
        // with per-cell divisions, which paced the whole pipeline).
        const uint64_t pol = ptx::l2_evict_first_policy();
        const bool tr = trc != nullptr;
        const int ua = range_lo(a.U, a.W, blockIdx.x), ub = range_lo(a.U, a.W, blockIdx.x + 1);
        const int nc = ub - ua, pre = nc < S ? nc : S;
        int gw = (int)(ua / Ul), ulw = ua - gw * Ul;          // weight cursor (layer, cell in layer)
        const uint32_t* src = a.packed[gw] + (a.rb0 * n_kc + ulw) * a.lay.cell_words;
        const uint32_t ring0 = ptx::smem_u32(ring);
        int s = 0;
        uint32_t r = 0;                                       // fills of stage s so far, mod 2
        auto issue_w = [&]() {                                // (elected lane) weight cell -> stage s
            ptx::mbar_arrive_expect_tx(full(s), kCellBytes);
            ptx::bulk_g2s_policy(ring0 + (uint32_t)s * kCellBytes, src, kCellBytes, full(s), pol);
        };
        auto advance_w = [&]() {
            if (++s == S) { s = 0; r ^= 1u; }
            src += a.lay.cell_words;
            if (++ulw == Ul && gw + 1 < a.G) {
                ulw = 0;
                ++gw;
                src = a.packed[gw] + a.rb0 * n_kc * a.lay.cell_words;
            }
        };
        for (int j = 0; j < pre; ++j) {
            if (ptx::elect_one()) issue_w();
            __syncwarp();
            advance_w();
        }
        ptx::pdl_wait();                                      // x~ is the previous kernel's output
        int gx = (int)(ua / Ul), ulx = ua - gx * Ul, KC = ulx % n_kc;   // x~ cursor
        const uint8_t* xsrc = a.xt[gx] + (size_t)KC * a.xcol_bytes;
        int xs = 0;                                           // x~ slot of cell j, its use parity
        uint32_t xph = 0;
        for (int j = 0; j < nc; ++j) {
            if (j >= XS) ptx::mbar_wait_sleep(xempty(xs), xph ^ 1u);
            const bool w = j >= pre;
            if (w && j >= S) ptx::mbar_wait_sleep(empty(s), r ^ 1u);
            if (ptx::elect_one()) {
                ptx::mbar_arrive_expect_tx(xfull(xs), a.xcol_bytes);
                ptx::bulk_g2s(xwin + (uint32_t)xs * a.xcol_bytes, xsrc, a.xcol_bytes, xfull(xs));
                if (w) issue_w();
            }
            __syncwarp();
            if (tr && lane == 0) utrace(9, j);
            if (w) advance_w();
            if (++xs == XS) { xs = 0; xph ^= 1u; }
            xsrc += a.xcol_bytes;
            if (++KC == n_kc) {
                KC = 0;
                xsrc = a.xt[gx];
            }
            if (++ulx == Ul && gx + 1 < a.G) {
                ulx = 0;
                ++gx;
                KC = 0;
                xsrc = a.xt[gx];
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer.  This warp shares its SM sub-partition with three decoder warps
        // and gets ~1/4 of its issue slots, so its per-cell path is kept short: every cell's metadata
        // (A buffer, x~ slot, barrier phases, segment flags) is computed up front by the 32 lanes into
        // an 8-byte shared-memory record, and the loop only reads two records, waits and issues the
        // MMAs of one or two cells (two when the second continues the first's row block).  (Traced:
        // the incremental-counter loop was ~130 SASS instructions per cell, ~650 cycles, and paced
        // the kernel.)
        const int ua = range_lo(a.U, a.W, blockIdx.x), ub = range_lo(a.U, a.W, blockIdx.x + 1);
        const int ncell = ub - ua;
        const uint32_t dstep = 2u * (uint32_t)a.BP;           // B descriptor step per MMA (16 K)
        const uint64_t cdesc0 = ptx::smem_desc_kmajor_noswizzle(xwin, a.lbo, a.sbo);
        const uint64_t cslot = (uint64_t)(a.xcol_bytes >> 4);  // descriptor start-address step per slot
        const bool tr = trc != nullptr;
        uint2* rec = reinterpret_cast<uint2*>(smem + a.off_rec);
        {
            const int KC0 = (ua - (ua / Ul) * Ul) % n_kc;     // row blocks are whole within a layer, so
            for (int jj = lane; jj < ncell; jj += 32) {       // the segment of cell jj is (KC0 + jj) / n_kc
                const int KC = (KC0 + jj) % n_kc, seg = (KC0 + jj) / n_kc;
                const int xs = jj % XS, lc = jj / kUG, ab = (jj % kUG) * kNBuf + (lc & (kNBuf - 1));
                const uint32_t first = (jj == 0 || KC == 0) ? 1u : 0u;
                const uint32_t meta = (uint32_t)xs | ((uint32_t)ab << 6) | ((uint32_t)((jj / XS) & 1) << 9) |
                                      ((uint32_t)((lc / kNBuf) & 1) << 10) | (first << 11) |
                                      ((jj + 1 == ncell || KC == n_kc - 1) ? 1u << 12 : 0u) |
                                      ((jj + XS < ncell) ? 1u << 13 : 0u) | ((uint32_t)(seg & 1) << 14) |
                                      ((first && seg >= 2) ? 1u << 15 : 0u) | ((uint32_t)(((seg >> 1) - 1) & 1) << 16);
                rec[jj] = make_uint2(tmem + kA0 + (uint32_t)ab * kACols, meta);
            }
            __syncwarp();
        }
        constexpr uint32_t kFirst = 1u << 11, kSegEnd = 1u << 12, kCommitX = 1u << 13, kDWait = 1u << 15;
        const uint32_t afull0 = bar0 + 8u * (2 * S), aempty0 = bar0 + 8u * (2 * S + kUG * kNBuf);
        uint32_t dcol = tmem;
        for (int jj = 0; jj < ncell;) {
            const uint2 r0 = rec[jj];
            const uint2 r1 = jj + 1 < ncell ? rec[jj + 1] : make_uint2(0u, kFirst);
            const bool pair = !(r1.y & kFirst);
            const bool first = (r0.y & kFirst) != 0;
            if (first) {
                const uint32_t d = (r0.y >> 14) & 1u;
                if (r0.y & kDWait) ptx::mbar_wait_sleep(dempty(d), (r0.y >> 16) & 1u);
                ptx::tc_fence_after();
                dcol = tmem + d * kD1;
            }
            const uint32_t xs0 = r0.y & 63u, ab0 = (r0.y >> 6) & 7u, xs1 = r1.y & 63u, ab1 = (r1.y >> 6) & 7u;
            ptx::mbar_wait_sleep(xfull(xs0), (r0.y >> 9) & 1u);
            ptx::mbar_wait_sleep(afull0 + 8u * ab0, (r0.y >> 10) & 1u);
            if (pair) {
                ptx::mbar_wait_sleep(xfull(xs1), (r1.y >> 9) & 1u);
                ptx::mbar_wait_sleep(afull0 + 8u * ab1, (r1.y >> 10) & 1u);
            }
            if (tr && lane == 0) {
                if (jj == 0) utrace(7, 1);
                utrace(4, jj);
            }
            ptx::tc_fence_after();
            const bool seg_end = ((pair ? r1.y : r0.y) & kSegEnd) != 0;
            if (ptx::elect_one()) {
                const uint64_t cd0 = cdesc0 + cslot * xs0;
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    ptx::umma_f16_ts(dcol, r0.x + 8u * (uint32_t)i, cd0 + (uint64_t)(dstep * (uint32_t)i), idesc,
                                     (first && i == 0) ? 0u : 1u);
                ptx::umma_commit(aempty0 + 8u * ab0);
                if (r0.y & kCommitX) ptx::umma_commit(xempty(xs0));
                if (pair) {
                    const uint64_t cd1 = cdesc0 + cslot * xs1;
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        ptx::umma_f16_ts(dcol, r1.x + 8u * (uint32_t)i, cd1 + (uint64_t)(dstep * (uint32_t)i), idesc, 1u);
                    ptx::umma_commit(aempty0 + 8u * ab1);
                    if (r1.y & kCommitX) ptx::umma_commit(xempty(xs1));
                }
                if (seg_end) ptx::umma_commit(dfull((r0.y >> 14) & 1u));
            }
            __syncwarp();
            if (tr && lane == 0) utrace(5, jj);
            jj += pair ? 2 : 1;
        }
    } else if (warp < 6) {
        // ================= epilogue warpgroup (warps 2-5: the four TMEM lane quadrants): D (thread =
        // row) -> y~ rows (whole row block) or a segment partial sum (split row block)
        __shared__ int s_last;
        const int q = warp & 3;
        const int R = 32 * q + lane;
        const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16);
        int seg = 0;
        for (int w = blockIdx.x; w < a.W; w += P) {
            const int ua = range_lo(a.U, a.W, w), ub = range_lo(a.U, a.W, w + 1);
            for (int RBv = ua / n_kc; RBv <= (ub - 1) / n_kc; ++RBv, ++seg) {
                const int d = seg & 1;
                ptx::mbar_wait_sleep(dfull(d), (uint32_t)((seg >> 1) & 1));
                if (R == 0) utrace(6, seg);
                ptx::tc_fence_after();
                const int g = RBv / a.nrb, RB = RBv - g * a.nrb;
                const int64_t row = (int64_t)RB * 128 + R;    // relative to the launch's first row
                const float sc = a.yscale[g];
                float* yo = a.yout[g] + row;
                const bool live = row < a.rows;
                const int w0 = range_of(a.U, a.W, RBv * n_kc), w1 = range_of(a.U, a.W, (RBv + 1) * n_kc - 1);
                const bool whole = w0 == w1;                   // the whole row block is this range's
                // split row block (stream-K): publish this range's partial sums; the last of the
                // w1 - w0 + 1 ranges to arrive adds them all in range order (fixed association)
                const int wf = range_of(a.U, a.W, g * Ul);
                float* segp = a.seg[g] + ((int64_t)(w0 - wf + RB) * a.BP) * 128 + R;
                float* dst = segp + (int64_t)(w - w0) * a.BP * 128;
#pragma unroll
                for (int cb = 0; cb < N; cb += 16) {          // 16 accumulator columns (batch rows) at a time
                    if (cb >= a.B) break;
                    uint32_t rr[16];
                    ptx::tmem_ld16(tl + (uint32_t)d * kD1 + (uint32_t)cb, rr);
                    ptx::tc_wait_ld();
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int bb = cb + i;
                        if (bb >= a.B) break;
                        const float v = __uint_as_float(rr[i]);
                        if (whole) {
                            if (live) yo[bb * a.ys] = v * sc;
                        } else {
                            dst[bb * 128] = v;
                        }
                    }
                }
                ptx::tc_fence_before();
                warp_arrive(dempty(d), lane);
                if (whole) continue;
                __threadfence();
                ptx::named_bar_sync(1, 128);
                if (R == 0) {
                    const int old = atomicAdd(a.ticket[g] + RB, 1);
                    const bool last = old == (int)(w1 - w0);
                    if (last) a.ticket[g][RB] = 0;             // every contributor has arrived: reset
                    s_last = last ? 1 : 0;
                }
                ptx::named_bar_sync(1, 128);
                if (s_last) {
                    __threadfence();
                    const int cnt = (int)(w1 - w0 + 1);
                    // four batch columns at a time with all their segment loads in flight: one L2 round
                    // trip per 4 columns (per column, it was 16 dependent round trips at B = 16: ncu had
                    // the batch-16 launch at 37 vs 22 us, warps parked at the exit barrier behind it)
                    for (int cb = 0; cb < a.B; cb += 4) {
                        float t[8][4];
#pragma unroll
                        for (int j = 0; j < 8; ++j)
#pragma unroll
                            for (int i = 0; i < 4; ++i)
                                t[j][i] = (j < cnt && cb + i < a.B) ? __ldcg(segp + (int64_t)j * a.BP * 128 + (cb + i) * 128) : 0.0f;
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            if (cb + i >= a.B) break;
                            float acc = t[0][i];                     // range order: a fixed association
#pragma unroll
                            for (int j = 1; j < 8; ++j)
                                if (j < cnt) acc += t[j][i];
                            for (int j = 8; j < cnt; ++j) acc += __ldcg(segp + (int64_t)j * a.BP * 128 + (cb + i) * 128);
                            if (live) yo[(cb + i) * a.ys] = acc * sc;
                        }
                    }
                }
            }
        }
    } else {
        // ================= decoder groups: cells jj = g, g + 3, ... of the CTA's cell sequence
        const int dw = warp - 6, g = dw >> 2, q = warp & 3;
        const int R = 32 * q + lane, I = R >> 4, rho = R & 15;
        const uint32_t ta_lane = tmem + ((uint32_t)(32 * q) << 16) + kA0;
        const uint32_t lut_lane = ptx::smem_u32(smem + kHdr) + 4u * (uint32_t)lane;
        int ncell = 0;
        for (int w = blockIdx.x; w < a.W; w += P) ncell += (int)(range_lo(a.U, a.W, w + 1) - range_lo(a.U, a.W, w));
        int lc = 0;
        for (int jj = g; jj < ncell; jj += kUG, ++lc) {
            const int s = jj % S;
            const uint32_t r = (uint32_t)((jj / S) & 1);
            const int b = lc & (kNBuf - 1), use = lc / kNBuf;
            const bool tr = lane == 0 && dw == 4 * g;
            ptx::mbar_wait_sleep(full(s), r);
            if (tr) utrace(1, jj);
            if (use > 0) ptx::mbar_wait_sleep(aempty(g, b), (uint32_t)((use - 1) & 1));
            if (tr) utrace(2, jj);
            ptx::tc_fence_after();
            const uint32_t* cellw = reinterpret_cast<const uint32_t*>(ring + (size_t)s * kCellBytes);
            const uint32_t ta = ta_lane + (uint32_t)(g * kNBuf + b) * kACols;
#pragma unroll 1
            for (int pp = 0; pp < 4; ++pp)                    // tile pairs of the cell
                udec::decode_pair<K, CODE, kImm>(cellw + (I * 4 + pp) * kTW * 2, rho, a.ca, lut_lane, ta + (uint32_t)pp * 16);
            warp_arrive(empty(s), lane);                      // the cell's stream words are read
            ptx::tc_wait_st();
            ptx::tc_fence_before();
            warp_arrive(afull(g, b), lane);
            if (tr) utrace(3, jj);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) utrace(7, 2);
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

struct UmmaPlan {
    int S, BP, N, XS;
    int64_t P, W, U;
    uint32_t xcol, off_ring, off_x, off_rec;
    size_t smem;
};

bool umma_plan(const Layout& lay, int code, int64_t B, int G, int64_t nrb, UmmaPlan* pl) {
    const bool hyb = code == QTIP_CODE_HYB;
    pl->BP = B <= 1 ? 1 : B <= 2 ? 2 : B <= 4 ? 4 : B <= 8 ? 8 : B <= 16 ? 16 : 64;
    pl->N = pl->BP <= 16 ? 16 : 64;
    pl->xcol = 128u * 2u * (uint32_t)pl->BP;                        // binary16 x~ (every code: 2 B per weight)
    const size_t cell = 2048u * (size_t)lay.k;
    const size_t lutb = hyb ? kLutBytes : 0;
    const size_t max_smem = 225 * 1024;                               // + the kernel's static shared memory
    pl->U = (int64_t)G * nrb * lay.n_kc;
    pl->P = std::min<int64_t>(num_sms(), pl->U);
    pl->W = pl->P;                                                    // one range per CTA, every range >= 1 cell
    const int S = umma_stages(lay.k, code);
    pl->S = S;
    const size_t pad = 512;                                           // the last slab's overlapping core-matrix rows
    const size_t recb = (size_t)(((pl->U + pl->P - 1) / pl->P + 1) * 8 + 15) & ~(size_t)15;   // MMA cell records
    const size_t fixed = kHdr + lutb + (size_t)S * cell + pad + recb;
    if (fixed >= max_smem) return false;
    const int64_t fit = (int64_t)((max_smem - fixed) / pl->xcol);
    pl->XS = (int)std::min<int64_t>(fit, kMaxXS);
    if (pl->XS < 2) return false;
    pl->off_ring = (uint32_t)(kHdr + lutb);
    pl->off_x = (uint32_t)(kHdr + lutb + (size_t)S * cell);
    pl->off_rec = (uint32_t)(pl->off_x + (size_t)pl->XS * pl->xcol + pad);
    pl->smem = pl->off_rec + recb;
    if ((uint64_t)pl->U * (uint64_t)(pl->W + 1) >= (1ull << 31)) return false;   // 32-bit index math in the kernel
    return pl->smem <= max_smem;
}

template <int K, int CODE, int N, bool kImm>
cudaError_t launch_umma_t(const UmmaArgs& a, const UmmaPlan& pl, cudaStream_t s) {
    auto kern = umma_gemv_kernel<K, CODE, N, kImm>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, dim3((unsigned)pl.P), dim3(kUThreads), pl.smem, s, a);
}

}  // namespace

bool umma_supported(const Layout& lay, int code, const CodeArgs& ca, int64_t B, int G) {
    if (B < 1 || B > 64 || lay.k < 2 || lay.k > 4 || G < 1 || G > kMaxGroup) return false;
    if (code == QTIP_CODE_HYB && (ca.Q != (int)kLutQ || ca.two_sign)) return false;
    UmmaPlan pl;
    return umma_plan(lay, code, B, G, lay.n_rb, &pl);
}

int umma_xt_mode(int code) { (void)code; return 7; }
int umma_batch_pad(int64_t B) { return B <= 1 ? 1 : B <= 2 ? 2 : B <= 4 ? 4 : B <= 8 ? 8 : B <= 16 ? 16 : 64; }

size_t umma_seg_floats(const Layout& lay, int code, int64_t B) {
    // segments of one layer for any group size: (W + nrb) x BP x 128
    size_t best = 0;
    for (int G = 1; G <= kMaxGroup; ++G) {
        UmmaPlan pl;
        if (!umma_plan(lay, code, B, G, lay.n_rb, &pl)) continue;
        best = std::max(best, (size_t)(pl.W + lay.n_rb) * pl.BP * 128);
    }
    return best;
}

cudaError_t launch_umma(const Layout& lay, int code, const CodeArgs& ca, int G, const void* const* packed,
                        const uint16_t* lut, const void* const* xt, float* const* seg, int* const* ticket,
                        float* const* yout, const float* yscale, int64_t ys, int64_t rows, int64_t B, int64_t rb0,
                        int64_t rb1, cudaStream_t s) {
    UmmaPlan pl;
    const int64_t nrb = rb1 - rb0;
    if (!umma_plan(lay, code, B, G, nrb, &pl)) return cudaErrorInvalidConfiguration;
    UmmaArgs a{};
    const float cf = (code == QTIP_CODE_1MAD) ? 5.0f / 739.0f : 1.0f;      // 1/147.8 for 1MAD (reading R6)
    for (int g = 0; g < G; ++g) {
        a.packed[g] = (const uint32_t*)packed[g];
        a.xt[g] = (const uint8_t*)xt[g];
        a.seg[g] = seg[g];
        a.ticket[g] = ticket[g];
        a.yout[g] = yout[g];
        a.yscale[g] = yscale[g] * cf;
    }
    a.ys = ys;
    a.rows = rows;
    a.lut = (const uint32_t*)lut;
    a.lay = lay;
    a.ca = ca;
    a.G = G;
    a.rb0 = rb0;
    a.nrb = (int)nrb;
    a.U = (int)pl.U;
    a.W = (int)pl.W;
    a.B = (int)B;
    a.BP = pl.BP;
    a.code_factor = cf;
    a.off_ring = pl.off_ring;
    a.off_x = pl.off_x;
    a.off_rec = pl.off_rec;
    a.xcol_bytes = pl.xcol;
    a.XS = pl.XS;
    a.lbo = 16u * (uint32_t)pl.BP;
    a.sbo = 128u;
    const bool imm = code != QTIP_CODE_HYB && lay.k == 2 &&
                     ca.a == (code == QTIP_CODE_1MAD ? 34038481u : 89226354u) &&
                     ca.b == (code == QTIP_CODE_1MAD ? 76625530u : 64248484u);
    cudaError_t e = cudaErrorInvalidValue;
#define QTIP_U_CASE(KK, CC, NN, II) \
    if (lay.k == KK && code == CC && pl.N == NN && imm == II) e = launch_umma_t<KK, CC, NN, II>(a, pl, s);
    QTIP_U_CASE(2, QTIP_CODE_3INST, 16, true) QTIP_U_CASE(2, QTIP_CODE_3INST, 64, true)
    QTIP_U_CASE(2, QTIP_CODE_1MAD, 16, true) QTIP_U_CASE(2, QTIP_CODE_1MAD, 64, true)
    QTIP_U_CASE(2, QTIP_CODE_3INST, 16, false) QTIP_U_CASE(2, QTIP_CODE_3INST, 64, false)
    QTIP_U_CASE(2, QTIP_CODE_1MAD, 16, false) QTIP_U_CASE(2, QTIP_CODE_1MAD, 64, false)
    QTIP_U_CASE(3, QTIP_CODE_3INST, 16, false) QTIP_U_CASE(3, QTIP_CODE_3INST, 64, false)
    QTIP_U_CASE(3, QTIP_CODE_1MAD, 16, false) QTIP_U_CASE(3, QTIP_CODE_1MAD, 64, false)
    QTIP_U_CASE(4, QTIP_CODE_3INST, 16, false) QTIP_U_CASE(4, QTIP_CODE_3INST, 64, false)
    QTIP_U_CASE(4, QTIP_CODE_1MAD, 16, false) QTIP_U_CASE(4, QTIP_CODE_1MAD, 64, false)
    QTIP_U_CASE(2, QTIP_CODE_HYB, 16, false) QTIP_U_CASE(2, QTIP_CODE_HYB, 64, false)
    QTIP_U_CASE(3, QTIP_CODE_HYB, 16, false) QTIP_U_CASE(3, QTIP_CODE_HYB, 64, false)
    QTIP_U_CASE(4, QTIP_CODE_HYB, 16, false) QTIP_U_CASE(4, QTIP_CODE_HYB, 64, false)
#undef QTIP_U_CASE
    count_launch(1);
    return e;
}

}  // namespace qtip

extern "C" int qtip_internal_set_umma_trace_cta(int cta) {
    return (int)cudaMemcpyToSymbol(qtip::g_umma_trace_cta, &cta, sizeof(cta));
}

extern "C" int qtip_internal_set_umma_trace(void* dptr) {
    unsigned long long* p = (unsigned long long*)dptr;
    return (int)cudaMemcpyToSymbol(qtip::g_umma_trace, &p, sizeof(p));
}
