// k_layer.cu -- the whole QTIP layer y = scale * S_m H_m^T W~ H_n S_n x in ONE
// persistent launch (impl 5): RHT-in, fused trellis-decode GEMV, split reduction and RHT-out,
// separated by in-kernel grid barriers instead of kernel boundaries.
//
// Grid: one 512-thread CTA per SM (all co-resident; grid barriers are self-resetting counters in
// the caller's zero-initialised workspace, with a 4 s watchdog that traps instead of hanging).
//
//   prologue   every warp requests its first S weight chunks (cp.async.bulk into a private ring);
//              the packed stream does not depend on the previous kernel, so this runs before the
//              PDL wait and overlaps the previous layer's tail.
//   x~         n = 2^a: every CTA computes the whole x~ = H_n S_n x / sqrt(n) itself (fp32 FWHT in
//              shared memory, register radix-8 passes) and keeps it resident in shared memory as
//              binary16 in mma.sync B-fragment order -- no barrier.  n = b 2^a, b > 1 (Paley
//              factor): every CTA does the Sylvester part, computes its slice of the dense H_b
//              mixing, publishes it, grid barrier, then loads all of x~.
//   GEMV       the launch's tile rows are cut into fixed "units" of U tile pairs (32 columns each)
//              along a row; unit partial sums (16 rows x B) come from one warp's register MMA
//              accumulation in a fixed order.  CTA c owns the contiguous unit range
//              [c T / P, (c+1) T / P) in row-major order, its warps take units round-robin.
//              Row sums are always (((p_0 + p_1) + p_2) + ...) over the row's units, so every
//              row's arithmetic depends on n only (a row shard equals the full call bit for bit).
//   reduce     rows whose units all lie in this CTA are summed in shared memory -> y~ (global);
//              rows shared with a neighbour CTA publish their unit partials; grid barrier.
//   RHT-out    every CTA assembles all of y~, runs the Sylvester FWHT, and writes its slice of
//              y = scale * S_m (H_m^T y~) / sqrt(m) (dense H_b^T mixing of its slice for b > 1).
//              Without RHT-out the owner of a row's last unit finishes the shared rows.
#include <algorithm>
#include <cmath>

#include "internal.h"
#include "fwht.cuh"
#include "mma_tile.cuh"
#include "tc.cuh"

namespace qtip {
namespace {

using namespace mma;
using namespace fw;

constexpr int kLWarps = 16;
constexpr int kLThreads = 32 * kLWarps;
constexpr int kLMaxStages = 16;
constexpr int kMixChunk = 256;               // outputs per dense-mixing round

struct LayerArgs {
    const uint32_t* packed;
    Layout lay;
    CodeArgs ca;
    const uint32_t* lut;
    const float* x;                          // [B][n]
    const uint8_t* sign_n;
    const uint8_t* sign_m;
    float scale, code_factor;
    float* y;                                // y[b * y_stride + (i - row_lo)]
    int64_t y_stride, row_lo, row_hi;
    int B;
    int rht_in, rht_out, xt_ready, coop;     // coop: x~ through global memory + a grid barrier
    int nb, na, mb, ma;                      // n = nb 2^na, m = mb 2^ma
    const uint32_t* hb_n;                    // H_nb bit rows (nb > 1)
    const uint32_t* hbt_m;                   // H_mb^T bit rows (mb > 1)
    uint32_t* xt_g;                          // x~ in fragment order, [B][row_words] words
    int64_t row_words;                       // n_pad (K-doubled codes) or n_pad / 2 (HYB)
    float* ybuf;                             // [B][m_pad] completed y~ rows
    float* gpart;                            // [B][m_pad][n_units] unit partials of shared rows
    unsigned* bar;                           // grid barrier {count at [0], generation at [32]}
    int64_t tile_row0;                       // first tile row of the launch
    int64_t T;                               // units in the launch
    int n_units, U, CP;                      // units per tile row, tile pairs per unit / chunk
    int stages;
    int max_units_cta;
    int part_smem;                           // unit partials in shared memory (else in gpart)
    uint32_t off_ring, off_x, off_v, off_red, off_out, off_outred, off_scr, off_lut;
    int finishers;                           // rows mode: CTAs (last arrivals) that run the RHT-out
    int debug;                               // knob 2: bit 0 = run the fast x~ phase twice (cold/warm probe)
    // grouped launch (G > 1): G layers of identical shape, CTAs [gcta0[g], gcta0[g+1]) run layer g
    // (rows mode, x~ ready, no RHT phases); the per-layer pointers replace the fields above
    int G;
    int gcta0[kMaxGroup + 1];
    const uint32_t* gpacked[kMaxGroup];
    uint32_t* gxt[kMaxGroup];
    float* gy[kMaxGroup];
    float gscale[kMaxGroup];
    float* ggpart[kMaxGroup];
    unsigned* gbar[kMaxGroup];
    const uint32_t* glut[kMaxGroup];
};

__device__ unsigned long long* g_layer_trace = nullptr;
__device__ int g_layer_trace_cap = 0;

// Phase timeline (debug): per CTA %globaltimer marks [0] entry, [1] PDL wait released, [2] input
// staged, [3] FWHT-in, [4] x~ ready, [5] GEMV done, [6] in-CTA reduction (+ barrier 1), [7] shared
// rows, [8] barrier 2, [9] y~ staged, [10] FWHT-out, [11] exit; records of 14 words
// {tag 5, blockIdx, t0..t11} after a u64 record counter.
constexpr int kMarks = 12;
__shared__ unsigned long long g_trs[kMarks];
__shared__ int g_trclk;                      // debug bit 4: SM clock64 marks (phase durations in cycles)
__device__ __forceinline__ void trace_mark(bool on, int i) {
    if (on && threadIdx.x == 0) {
        unsigned long long t;
        if (g_trclk) t = clock64();
        else asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_trs[i] = t;
    }
}

__device__ __forceinline__ int swz(int i) { return i ^ (((i >> 6) & 3) << 3); }

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Grid barrier: arrival counter and generation word on different 128-B lines (bar[0], bar[32]);
// the last arrival resets the counter and bumps the generation, the others poll the generation
// with relaxed loads and fence once.  The counter is 0 between barriers (zero-initialised
// workspace); a 4 s watchdog traps instead of hanging if a CTA is missing.
// Measured variants: scripts/gridbar_microbench.cu.
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned P) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned* cnt = bar;
        unsigned* gen = bar + 32;
        unsigned g, old;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(gen) : "memory");
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
        if (old == P - 1) {
            asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(cnt) : "memory");
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(g + 1) : "memory");
        } else {
            const uint64_t t0 = gtimer();
            while (true) {
                unsigned v;
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gen) : "memory");
                if (v != g) break;
                if (gtimer() - t0 > 4000000000ull) __trap();
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
    }
    __syncthreads();
}

// The canonical sum of a row's unit partials p_u (u < nu, element stride st): lane l adds
// p_l, p_{l+32}, ... in order, then a fixed xor butterfly over the lanes (every lane ends with
// the same bits).  Used for every row, in-CTA or shared, so a row's value depends on n only.
template <bool kGlobal>
__device__ __forceinline__ float warp_row_sum(const float* p, int64_t st, int nu) {
    const int lane = threadIdx.x & 31;
    float t = 0.0f;
#pragma unroll 1
    for (int u = lane; u < nu; u += 32) t += kGlobal ? __ldcg(p + u * st) : p[u * st];   // compact: cold code
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    return t;
}

// The same canonical sum (bit for bit: lane-strided partial sums, then the xor-butterfly tree seen
// from lane 0) computed by ONE thread, so a CTA reduces many rows in parallel (one thread per row)
// instead of one warp per row.
__device__ __forceinline__ float thread_row_sum(const float* p, int st, int nu) {
    float s[32];
#pragma unroll
    for (int l = 0; l < 32; ++l) s[l] = 0.0f;
#pragma unroll 1
    for (int u0 = 0; u0 < nu; u0 += 32) {
        // all loads first (clamped in range, branch-free): one latency per chunk, not 32
        const float* q = p + u0 * st;
        const int last = nu - 1 - u0;
        float v[32];
#pragma unroll
        for (int l = 0; l < 32; ++l) v[l] = q[(l < last ? l : last) * st];
#pragma unroll
        for (int l = 0; l < 32; ++l) s[l] = l <= last ? s[l] + v[l] : s[l];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1)
#pragma unroll
        for (int l = 0; l < o; ++l) s[l] += s[l + o];
    return s[0];
}

// One radix-2^R pass of the Walsh-Hadamard butterflies on index bits [p, p + R) of v (swizzled).
template <int R>
__device__ __forceinline__ void fwht_pass(float* v, int len, int p) {
    constexpr int G = 1 << R;
    const int ng = len >> R;
    const int pm = (1 << p) - 1;
    for (int gi = threadIdx.x; gi < ng; gi += kLThreads) {
        const int base = (gi & pm) | ((gi >> p) << (p + R));
        float u[G];
        bool vec = false;
        if constexpr (R == 3) {
            if (p == 0) {                                            // 8 contiguous floats: 2 x LDS.128
                const float4* q = reinterpret_cast<const float4*>(v + swz(base));
                const float4 a = q[0], b = q[1];
                u[0] = a.x; u[1] = a.y; u[2] = a.z; u[3] = a.w; u[4] = b.x; u[5] = b.y; u[6] = b.z; u[7] = b.w;
                vec = true;
            }
        }
        if (!vec) {
#pragma unroll
            for (int j = 0; j < G; ++j) u[j] = v[swz(base + (j << p))];
        }
#pragma unroll
        for (int h = 1; h < G; h <<= 1)
#pragma unroll
            for (int j = 0; j < G; ++j)
                if (!(j & h)) {
                    const float a = u[j], b = u[j | h];
                    u[j] = a + b;
                    u[j | h] = a - b;
                }
        if constexpr (R == 3) {
            if (vec) {
                float4* q = reinterpret_cast<float4*>(v + swz(base));
                q[0] = make_float4(u[0], u[1], u[2], u[3]);
                q[1] = make_float4(u[4], u[5], u[6], u[7]);
            }
        }
        if (!vec) {
#pragma unroll
            for (int j = 0; j < G; ++j) v[swz(base + (j << p))] = u[j];
        }
    }
}

// Sylvester transform along index bits [0, a) of every 2^a block of v[0, len) (no scaling).
__device__ __noinline__ void cta_fwht(float* v, int len, int a) {
    for (int p = 0; p < a;) {
        const int r = min(3, a - p);
        if (r == 3) fwht_pass<3>(v, len, p);
        else if (r == 2) fwht_pass<2>(v, len, p);
        else fwht_pass<1>(v, len, p);
        __syncthreads();
        p += r;
    }
}

// Dense Paley-factor mixing of flat outputs [f0, f1) (f = bt * len + i_b 2^a + i_a):
// out = sum_jb Hbits[i_b][jb] v[bt][jb][i_a]; warps split jb, partials added in warp order.
// emit(f, value) is called once per output by threads 0 .. kMixChunk-1.
template <typename Emit>
__device__ __noinline__ void dense_mix(const float* v, int len, int b, int a, const uint32_t* __restrict__ hbits,
                                       int f0, int f1, float* red, Emit emit) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wpr = (b + 31) >> 5;
    const int jlo = b * warp / kLWarps, jhi = b * (warp + 1) / kLWarps;
    const int am = (1 << a) - 1;
    for (int c0 = f0; c0 < f1; c0 += kMixChunk) {
        const int cnt = f1 - c0 < kMixChunk ? f1 - c0 : kMixChunk;
#pragma unroll 1
        for (int e = 0; e < kMixChunk / 32; ++e) {
            const int fl = lane + 32 * e;
            float s = 0.0f;
            if (fl < cnt) {
                const int f = c0 + fl;
                const int bt = f / len, i = f - bt * len;
                const int ib = i >> a, ia = i & am;
                const uint32_t* hr = hbits + ib * wpr;
                for (int jb = jlo; jb < jhi; ++jb) {
                    const float x = v[swz(bt * len + (jb << a) + ia)];
                    const uint32_t neg = (__ldg(hr + (jb >> 5)) >> (jb & 31)) & 1u;
                    s += neg ? -x : x;
                }
            }
            red[warp * kMixChunk + fl] = s;
        }
        __syncthreads();
        if (threadIdx.x < cnt) {
            float s = 0.0f;
#pragma unroll
            for (int w = 0; w < kLWarps; ++w) s += red[w * kMixChunk + threadIdx.x];
            emit(c0 + threadIdx.x, s);
        }
        __syncthreads();
    }
}

__device__ __forceinline__ uint32_t sgn(const uint8_t* __restrict__ s, int64_t i) {
    return (__ldg(s + (i >> 3)) >> (i & 7)) & 1u;
}

// vb[swz(bt * dst_stride + e)] = S[e] src[bt * src_stride + e] for bt < B, e < len (fp32 in global
// memory, possibly the previous kernel's output: L2 loads); e in [len, dst_stride) is zero-filled.
// Four 16-B loads in flight per thread.
__device__ __noinline__ void stage_input(float* vb, int dst_stride, const float* src, int64_t src_stride,
                                         const uint8_t* __restrict__ sign, int B, int len) {
    const int qpr = dst_stride >> 2, nq = B * qpr;                  // len, dst_stride multiples of 4
    for (int q0 = threadIdx.x; q0 < nq; q0 += 4 * kLThreads) {
        float4 v[4];
        uint32_t sb[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int q = q0 + j * kLThreads;
            v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
            sb[j] = 0u;
            if (q < nq) {
                const int bt = q / qpr, e = 4 * (q - bt * qpr);
                if (e < len) {
                    v[j] = __ldcg(reinterpret_cast<const float4*>(src + bt * src_stride + e));
                    if (sign) sb[j] = (uint32_t)__ldg(sign + (e >> 3)) >> (e & 7);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int q = q0 + j * kLThreads;
            if (q < nq) {
                float4 w = v[j];
                if (sb[j] & 1u) w.x = -w.x;
                if (sb[j] & 2u) w.y = -w.y;
                if (sb[j] & 4u) w.z = -w.z;
                if (sb[j] & 8u) w.w = -w.w;
                *reinterpret_cast<float4*>(vb + swz(4 * q)) = w;
            }
        }
    }
}

// x~ element (bt, e) -> binary16 in B-fragment order (the RHT kernel's out_mode 3 / 4, or 5 with kSwap).
template <bool kHyb, bool kSwap = false>
__device__ __forceinline__ void put_xt(uint32_t* xs, int64_t row_words, int bt, int64_t e, float v) {
    const uint32_t h = __half_as_ushort(__float2half_rn(v));
    const int64_t tile = e >> 4;
    const int c = (int)(e & 15);
    if constexpr (!kHyb) {
        const int t = (c & 7) >> 1, q = ((c & 1) << 1) | (c >> 3);
        xs[bt * row_words + tile * 16 + 4 * t + q] = h | (h << 16);
    } else {
        const int j = c >> 1;
        const int64_t w = tile * 8 + 2 * (j & 3) + (j >> 2);
        reinterpret_cast<uint16_t*>(xs + bt * row_words)[2 * w + ((c & 1) ^ (kSwap ? 1 : 0))] = (uint16_t)h;
    }
}

__device__ __noinline__ void rht_out_phase(const LayerArgs& args, uint8_t* smem, int64_t c, int64_t P, bool tr);

// 16 warps, up to 128 registers: exactly one CTA of this kernel per SM (the grid is one CTA per
// SM, and two would not fit), while the small RHT kernels around it can still share the SM.
template <int K, int CODE, bool kImm>
__global__ void __launch_bounds__(kLThreads, 1) layer_kernel(const __grid_constant__ LayerArgs args) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr bool kHyb = CODE == QTIP_CODE_HYB;
    constexpr bool kHybFast = kHyb;                                // Q = 9 (layer_supported)
    constexpr int TW = 8 * K;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, tig = lane & 3;
    const int B = args.B, S = args.stages;
    int grp = 0;                                                    // layer of a grouped launch
    while (grp + 1 < args.G && (int)blockIdx.x >= args.gcta0[grp + 1]) ++grp;
    const bool grouped = args.G > 1;
    const int64_t P = grouped ? args.gcta0[grp + 1] - args.gcta0[grp] : (int64_t)gridDim.x;
    const int64_t c = grouped ? (int64_t)blockIdx.x - args.gcta0[grp] : (int64_t)blockIdx.x;
    const uint32_t* const a_packed = grouped ? args.gpacked[grp] : args.packed;
    uint32_t* const a_xt = grouped ? args.gxt[grp] : args.xt_g;
    float* const a_y = grouped ? args.gy[grp] : args.y;
    const float a_scale = grouped ? args.gscale[grp] : args.scale;
    float* const a_gpart = grouped ? args.ggpart[grp] : args.gpart;
    unsigned* const a_bar = grouped ? args.gbar[grp] : args.bar;
    const uint32_t* const a_lut = grouped ? args.glut[grp] : args.lut;
    const int64_t n = args.lay.n, m = args.lay.m, n_kc = args.lay.n_kc, m_pad = args.lay.m_pad;
    const int n_units = args.n_units, U = args.U, CP = args.CP;
    const int64_t T = args.T;
    // rows mode (launch tile rows >= CTAs): CTA c owns whole tile rows [c R / P, (c+1) R / P), no row
    // is shared; else CTA c owns units [c T / P, (c+1) T / P) and rows may straddle CTAs
    const int64_t R = T / n_units;
    const bool rows_mode = R >= P;
    const int64_t L0 = rows_mode ? (c * R / P) * n_units : c * T / P;
    const int64_t L1 = rows_mode ? ((c + 1) * R / P) * n_units : (c + 1) * T / P;
    const uint32_t chunk_bytes = 256u * K;                          // one cell's tile row
    const int n_pairs = (int)(n_kc * 4);

    const bool tr = g_layer_trace != nullptr;
    if (tr && threadIdx.x == 0) g_trclk = (args.debug & 4) != 0;
    if (tr && threadIdx.x == 0)
        for (int q = 0; q < kMarks; ++q) g_trs[q] = 0;
    trace_mark(tr, 0);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem) + warp * kLMaxStages;
    float* part = reinterpret_cast<float*>(smem + 8 * kLWarps * kLMaxStages);   // [unit - L0][16][B]
    uint8_t* ring = smem + args.off_ring + (size_t)warp * S * chunk_bytes;
    uint32_t* xs = reinterpret_cast<uint32_t*>(smem + args.off_x);
    float* vb = reinterpret_cast<float*>(smem + args.off_v);
    float* red = reinterpret_cast<float*>(smem + args.off_red);

    // ---- warp's units L = L0 + warp + j W (one unit = one ring chunk = one cell's tile row: 4 tile
    //      pairs, 128 columns, 256 k bytes); 32-bit incremental (row, unit-in-row) iterators
    struct UnitIt {
        int L, Ir, u;                                               // launch unit, tile row, unit in row
        __device__ __forceinline__ void step(int n_units) {
            L += kLWarps;
            u += kLWarps;
            if (u >= n_units) {                                     // n_units >= 16: at most one wrap
                u -= n_units;
                ++Ir;
                while (u >= n_units) { u -= n_units; ++Ir; }        // narrow layers only
            }
        }
    };
    const int L0i = (int)L0, L1i = (int)L1;
    // the end-of-launch reduction's row range, computed here (its integer divisions off the tail)
    int Ia = 0, nrow_items = 0;
    if (L1 > L0) {
        Ia = L0i / n_units;
        nrow_items = ((L1i - 1) / n_units - Ia + 1) * kTile * B;
    }
    UnitIt first{L0i + warp, (L0i + warp) / n_units, (L0i + warp) % n_units};
    // Weight chunks are fetched by the whole warp with 16-byte cp.async (LDGSTS) into its ring stage,
    // each lane arriving on the stage's mbarrier when its copies land.  Measured: one
    // cp.async.bulk per 512-B chunk (lane 0) capped the steady state at 8.6 weights/clk/SM
    // (scripts/gemv_rate.py); per-lane copies keep many more requests in flight.
    const uint64_t wpol = ptx::l2_evict_first_policy();
    auto issue = [&](const UnitIt& it, int st) {
        const int I = (int)args.tile_row0 + it.Ir;
        const uint32_t bar = ptx::smem_u32(full + st);
        const uint8_t* src = reinterpret_cast<const uint8_t*>(
            a_packed + ((int64_t)(I >> 3) * n_kc + it.u) * (512 * K) + (I & 7) * (64 * K));
        const uint32_t dst = ptx::smem_u32(ring + (size_t)st * chunk_bytes);
#pragma unroll
        for (int q = 0; q < (16 * K + 31) / 32; ++q) {               // 16 K pieces of 16 B
            const int piece = lane + 32 * q;
            if (piece < 16 * K) ptx::cp_async16_stream(dst + 16 * piece, src + 16 * piece, wpol);
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
    };
    UnitIt iit = first;                                             // issue-side iterator (all lanes)
    int ist = 0;
    auto issue_next = [&]() {
        if (iit.L >= L1i) return;
        issue(iit, ist);
        if (++ist == S) ist = 0;
        iit.step(n_units);
    };
    if (lane == 0) {
        for (int st = 0; st < S; ++st) ptx::mbar_init(ptx::smem_u32(full + st), 32);
        ptx::fence_mbar_init();
    }
    __syncwarp();
    for (int st = 0; st < S; ++st) issue_next();
    __syncwarp();
    trace_mark(tr, 7);

    if constexpr (kHybFast) {                                       // 32-way replicated LUT, words (c0 << 16) | c1
        uint32_t* lsm = reinterpret_cast<uint32_t*>(smem + args.off_lut);
        for (int i = threadIdx.x; i < (512 << 5); i += kLThreads) {
            const uint32_t v = __ldg(a_lut + (i >> 5));
            lsm[i] = (v << 16) | (v >> 16);
        }
    }
    ptx::pdl_wait();                                                // x may be the previous kernel's output
    trace_mark(tr, 1);

    // ---------------------------------------------------------------- x~
    const int64_t rw = args.row_words;
    // x~ row stride in shared memory: padded (64 B / HYB 32 B) when x~ is copied in from the workspace
    // and B > 1, so a B-fragment load's batch rows spread over all bank groups
    const int xrs = ((args.xt_ready || args.coop) && B > 1) ? (int)rw + (kHyb ? 8 : 16) : (int)rw;
    const int64_t n_pad = args.lay.n_pad;
    if (args.xt_ready || args.coop) {
        if (args.coop && !args.xt_ready) {
            // Sylvester part of every block (redundant), then this CTA's slice of the H_b mixing
            const int len = (int)n;
            stage_input(vb, len, args.x, n, args.rht_in ? args.sign_n : nullptr, B, len);
            __syncthreads();
            cta_fwht(vb, B * len, args.na);
            const float rs = rsqrtf((float)n);
            const int64_t F = (int64_t)B * len;
            uint32_t* xg = a_xt;
            dense_mix(vb, len, args.nb, args.na, args.hb_n, (int)(c * F / P), (int)((c + 1) * F / P), red,
                      [=](int f, float s) { put_xt<kHyb, kHybFast>(xg, rw, f / len, f % len, s * rs); });
            if (c == 0) {                                           // zero padding columns [n, n_pad)
                const int pad = (int)(n_pad - n);
                for (int i = threadIdx.x; i < B * pad; i += kLThreads)
                    put_xt<kHyb, kHybFast>(a_xt, rw, i / pad, n + i % pad, 0.0f);
            }
            grid_sync(a_bar, (unsigned)P);
        }
        const int words = (int)(B * rw), rq = (int)(rw / 4), xq = xrs / 4;
        for (int i = threadIdx.x; i < words / 4; i += kLThreads) {          // rows at the padded stride
            const int row = i / rq;
            reinterpret_cast<uint4*>(xs)[row * xq + (i - row * rq)] = __ldcg(reinterpret_cast<const uint4*>(a_xt) + i);
        }
    } else {
        const int len = (int)n, np = (int)n_pad;
        const int Ef = args.rht_in ? fwht_fast_E(n, args.na, kLThreads) : 0;
        if (Ef) {
            // register / shuffle FWHT per batch row straight from global x; fragment-order x~ out
            float* scr = reinterpret_cast<float*>(smem + args.off_scr);
            const float rs = rsqrtf((float)n);
            for (int rep = 0; rep < 1 + (args.debug & 1); ++rep) {
            for (int bt = 0; bt < B; ++bt) {
                auto run = [&](auto EE) {
                    constexpr int E = decltype(EE)::value;
                    float v[E];
                    const int T = len / E;
                    uint32_t sb = 0;
                    if ((int)threadIdx.x < T) {
                        const int e0 = threadIdx.x * E;
                        sb = (uint32_t)__ldg(reinterpret_cast<const uint16_t*>(args.sign_n) + (e0 >> 4)) >> (e0 & 15);
#pragma unroll
                        for (int e = 0; e < E; e += 4) {
                            const float4 q = __ldcg(reinterpret_cast<const float4*>(args.x + bt * n + e0 + e));
                            v[e] = q.x; v[e + 1] = q.y; v[e + 2] = q.z; v[e + 3] = q.w;
                        }
#pragma unroll
                        for (int e = 0; e < E; ++e)
                            if ((sb >> e) & 1u) v[e] = -v[e];
                    } else {
#pragma unroll
                        for (int e = 0; e < E; ++e) v[e] = 0.0f;
                    }
                    trace_mark(tr, 2);
                    const int i0 = fwht_fast<E>(v, args.na, scr);
                    trace_mark(tr, 3);
                    park_tiles<E>(v, i0, args.na, scr);
                    const int wpt = kHyb ? 8 : 16;                  // x~ words per tile
                    for (int tile = threadIdx.x; tile < (len >> 4); tile += kLThreads) {
                        float o[16];
                        tile_read<E>(scr, tile, o);
#pragma unroll
                        for (int q = 0; q < 16; ++q) o[q] *= rs;
                        put_tile<kHyb, kHybFast>(xs + bt * rw + tile * wpt, o);
                        if (c == 0 && a_xt) put_tile<kHyb, kHybFast>(a_xt + bt * rw + tile * wpt, o);
                    }
                    __syncthreads();                                // scr reused by the next batch row
                };
                if (Ef == 4) run(std::integral_constant<int, 4>{});
                else if (Ef == 8) run(std::integral_constant<int, 8>{});
                else run(std::integral_constant<int, 16>{});
            }
            __syncthreads();
            }
            for (int i = threadIdx.x; i < B * (np - len); i += kLThreads) {   // zero padding columns
                const int bt = i / (np - len);
                put_xt<kHyb, kHybFast>(xs, rw, bt, len + i - bt * (np - len), 0.0f);
            }
        } else {
        // x~ in place: vb (fp32, batch stride n_pad, zero padded) and xs share memory; each thread
        // converts one 16-column tile, all reads of a chunk of tiles precede its writes (a tile's
        // data and its fragment words stay inside one 32-element swizzle block)
        stage_input(vb, np, args.x, n, args.rht_in ? args.sign_n : nullptr, B, len);
        __syncthreads();
        trace_mark(tr, 2);
        float rs = 1.0f;
        if (args.rht_in) {
            cta_fwht(vb, B * np, args.na);
            rs = rsqrtf((float)n);
        }
        trace_mark(tr, 3);
        const int tpr = np >> 4, ntiles = B * tpr;
        for (int t0 = 0; t0 < ntiles; t0 += kLThreads) {
            const int t = t0 + threadIdx.x;
            float v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = t < ntiles ? vb[swz(16 * t + q)] * rs : 0.0f;
            __syncthreads();
            if (t < ntiles) {
                const int bt = t / tpr, e0 = 16 * (t - bt * tpr);
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    put_xt<kHyb, kHybFast>(xs, rw, bt, e0 + q, v[q]);
                    if (c == 0 && a_xt) put_xt<kHyb, kHybFast>(a_xt, rw, bt, e0 + q, v[q]);   // QTIP_XT_READY reuse
                }
            }
            __syncthreads();
        }
        }
    }
    __syncthreads();
    trace_mark(tr, 4);
    const int pdl_at = (args.debug >> 3) & 3;                        // debug: 0 here, 1 after GEMV, 2 after reduction
    if (pdl_at == 0) ptx::pdl_launch_dependents();

    // ---------------------------------------------------------------- GEMV over the warp's units
    const CodeArgs ca = args.ca;
    const Lcg<CODE, kImm> lcg(ca);
    // B-fragment base of this lane (batch row g, K-slot group tig); lanes with g >= B read a zero
    // block instead (unit stride 0), so the loop has no predicated loads or zeroing
    __shared__ __align__(16) uint32_t zero_b[128];
    if (threadIdx.x < 128) zero_b[threadIdx.x] = 0u;
    __syncthreads();
    const bool bval = g < B;
    const uint32_t* xsl = bval ? xs + g * xrs + (kHyb ? 2 : 4) * tig : zero_b + (kHyb ? 2 : 4) * tig;
    const int ustride = bval ? (kHyb ? 64 : 128) : 0;
    const uint32_t* lut = a_lut;
    const uint32_t lut_lane = ptx::smem_u32(smem + args.off_lut) + 4u * lane;
    const mma::HybFastLane hl = mma::hyb_fast_lane(g, tig);
    const mma::HybFastLaneK<K> hlk = mma::hyb_fast_lane_k<K>(g, tig);
    const uint32_t full0 = ptx::smem_u32(full);
    const uint8_t* ring0 = ring;
    const uint32_t part_u32 = ptx::smem_u32(part);
    uint32_t poff[4];
    bool pok[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int b = 2 * tig + (e & 1), r = 2 * g + (e >> 1);
        pok[e] = b < B;
        poff[e] = (uint32_t)(r * B + (b < B ? b : 0)) * 4u;
    }
    auto run = [&](auto kPartSmem, auto kTwoSign) {
        constexpr bool kSmemPart = decltype(kPartSmem)::value;
        constexpr bool kTwo = decltype(kTwoSign)::value;
        float* const gpart = a_gpart;
        const int64_t row0 = args.tile_row0 * kTile;
        int st = 0;
        uint32_t phase = 0;
        for (UnitIt it = first; it.L < L1i; it.step(n_units)) {
            float acc[2][1][4] = {{{0.f, 0.f, 0.f, 0.f}}, {{0.f, 0.f, 0.f, 0.f}}};
            ptx::mbar_wait_sleep(full0 + 8 * st, phase);
            const uint32_t* chunk = reinterpret_cast<const uint32_t*>(ring0 + (size_t)st * chunk_bytes);
            const uint32_t* xu = xsl + ustride * it.u;              // x~ of the unit's 8 tile columns
            // all shared-memory operands of the unit are loaded up front (the decode then never waits
            // on LDS latency in the middle of a tile pair: short_scoreboard stalls in ncu)
            uint32_t bf[4][2][1][4];
#pragma unroll
            for (int pp = 0; pp < 4; ++pp)
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    if constexpr (!kHyb) {
                        const uint4 v = *reinterpret_cast<const uint4*>(xu + 16 * (2 * pp + t));
                        bf[pp][t][0][0] = v.x; bf[pp][t][0][1] = v.y; bf[pp][t][0][2] = v.z; bf[pp][t][0][3] = v.w;
                    } else {
                        const uint2 v = *reinterpret_cast<const uint2*>(xu + 8 * (2 * pp + t));
                        bf[pp][t][0][0] = v.x; bf[pp][t][0][1] = v.y; bf[pp][t][0][2] = bf[pp][t][0][3] = 0u;
                    }
                }
            if constexpr (K == 2 && !kHyb) {
                uint4 w01[4];
                uint2 w2[4];
#pragma unroll
                for (int pp = 0; pp < 4; ++pp) {
                    w01[pp] = *reinterpret_cast<const uint4*>(chunk + pp * TW * 2 + 2 * (2 * g));
                    w2[pp] = *reinterpret_cast<const uint2*>(chunk + pp * TW * 2 + 2 * ((2 * g + 2) & 15));
                }
#pragma unroll
                for (int pp = 0; pp < 4; ++pp)
                    tile_pair_k2_words<CODE, 1, kImm>(w01[pp], w2[pp], bf[pp], acc[pp & 1], tig, lcg, ca);
            } else {
#pragma unroll
                for (int pp = 0; pp < 4; ++pp) {
                    if constexpr (kHybFast && K == 4) tile_pair_hyb4<1, kTwo>(chunk + pp * TW * 2, bf[pp], acc[pp & 1], hl, lut_lane);
                    else if constexpr (kHybFast) tile_pair_hyb_k<K, 1, kTwo>(chunk + pp * TW * 2, bf[pp], acc[pp & 1], hlk, lut_lane);
                    else tile_pair<K, CODE, 1, kImm>(chunk + pp * TW * 2, bf[pp], acc[pp & 1], g, tig, lcg, ca, lut);
                }
            }
            __syncwarp();
            if (iit.L < L1i) issue_next();                           // refill (only if the ring was too small)
            if (++st == S) { st = 0; phase ^= 1u; }
            // acc[e] = D[MMA row g + 8 (e >> 1)][batch 2 tig + (e & 1)] <-> tile row 2g + (e >> 1);
            // branch-free predicated stores (lane-constant offsets and predicates)
            if constexpr (kSmemPart) {
                const uint32_t ub = part_u32 + (uint32_t)(it.L - L0i) * (uint32_t)(kTile * 4 * B);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float v = acc[0][0][e] + acc[1][0][e];
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p st.shared.f32 [%0], %1;\n\t}"
                                 ::"r"(ub + poff[e]), "f"(v), "r"((uint32_t)pok[e]) : "memory");
                }
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int b = 2 * tig + (e & 1), r = 2 * g + (e >> 1);
                    if (b < B) gpart[((int64_t)b * m_pad + row0 + it.Ir * kTile + r) * n_units + it.u] = acc[0][0][e] + acc[1][0][e];
                }
            }
        }
    };
    if (kHyb && ca.two_sign) {
        if (args.part_smem) run(std::true_type{}, std::integral_constant<bool, kHyb>{});
        else run(std::false_type{}, std::integral_constant<bool, kHyb>{});
    } else {
        if (args.part_smem) run(std::true_type{}, std::false_type{});
        else run(std::false_type{}, std::false_type{});
    }
    __syncthreads();
    trace_mark(tr, 5);
    if (pdl_at == 1) ptx::pdl_launch_dependents();

    // ---------------------------------------------------------------- reduction (warp per row)
    const bool rht_out = args.rht_out != 0;
    auto owner = [&](int64_t L) { return ((L + 1) * P - 1) / T; };    // unit mode: CTA whose range holds unit L
    auto finish = [&](int b, int64_t i, float s) {                    // s = the row's canonical sum
        s *= args.code_factor;
        if (rht_out) args.ybuf[b * m_pad + i] = s;
        else if (i >= args.row_lo && i < args.row_hi) a_y[b * args.y_stride + (i - args.row_lo)] = a_scale * s;
    };
    const int tile_row0 = (int)args.tile_row0;
    trace_mark(tr && rows_mode && !rht_out, 9);
    if (rows_mode) {
        // every row of this CTA is complete here: one thread per (row, batch) item
        for (int t = threadIdx.x; t < nrow_items; t += kLThreads) {
            const int tb = t / B, b = t - tb * B;
            const int Ir = Ia + (tb >> 4), r = tb & 15;
            const int i = (tile_row0 + Ir) * kTile + r;
            const int u0 = Ir * n_units;
            finish(b, i, args.part_smem ? thread_row_sum(part + ((u0 - L0i) * kTile + r) * B + b, kTile * B, n_units)
                                        : thread_row_sum(a_gpart + ((int64_t)b * m_pad + i) * n_units, 1, n_units));
        }
        nrow_items = 0;                                               // nothing left for the warp loop
    }
    for (int t = warp; t < nrow_items; t += kLWarps) {
        if (t == 0) trace_mark(tr && rows_mode && !rht_out, 10);
        const int tb = t / B, b = t - tb * B;
        const int Ir = Ia + (tb >> 4), r = tb & 15;
        const int i = (tile_row0 + Ir) * kTile + r;
        const int u0 = Ir * n_units;
        if (u0 >= L0i && u0 + n_units <= L1i) {                       // every unit in this CTA
            const float s = args.part_smem
                ? warp_row_sum<false>(part + ((u0 - L0i) * kTile + r) * B + b, kTile * B, n_units)
                : warp_row_sum<true>(a_gpart + ((int64_t)b * m_pad + i) * n_units, 1, n_units);
            if (t == 0) trace_mark(tr && rows_mode && !rht_out, 7);       // debug: first row's sum
            if (lane == 0) finish(b, i, s);
            if (t == 0) trace_mark(tr && rows_mode && !rht_out, 8);
        } else if (args.part_smem) {                                  // shared row: publish this CTA's units
            const int s_lo = L0i - u0 > 0 ? L0i - u0 : 0, s_hi = L1i - u0 < n_units ? L1i - u0 : n_units;
            for (int u = s_lo + lane; u < s_hi; u += 32)
                a_gpart[((int64_t)b * m_pad + i) * n_units + u] = part[((u0 + u - L0i) * kTile + r) * B + b];
        }
    }
    trace_mark(tr, 6);
    if (pdl_at == 2) ptx::pdl_launch_dependents();
    if (rows_mode) {
        // no shared rows.  RHT-out: every CTA takes a ticket after publishing its y~ rows; the last
        // `finishers` arrivals run the RHT-out (the very last one alone when m = 2^a), the others
        // exit at once and free their SM for the next launch (no grid barrier).
        if (rht_out) {
            __shared__ int s_ticket;
            const int G = args.finishers;
            __syncthreads();
            if (threadIdx.x == 0) {
                unsigned long long* cnt = reinterpret_cast<unsigned long long*>(a_bar + 64);
                unsigned long long old;
                __threadfence();
                asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(old) : "l"(cnt) : "memory");
                const int tk = (int)(old % (unsigned long long)P);
                s_ticket = tk;
                if (tk >= P - G && tk < P - 1) {                        // wait for the remaining arrivals
                    const unsigned long long target = (old / P + 1) * P;
                    const uint64_t t0 = gtimer();
                    while (true) {
                        unsigned long long v;
                        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(cnt) : "memory");
                        if (v >= target) break;
                        if (gtimer() - t0 > 4000000000ull) __trap();
                    }
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                }
            }
            __syncthreads();
            const int tk = s_ticket;
            trace_mark(tr, 8);
            if (tk >= P - G) rht_out_phase(args, smem, tk - (P - G), G, tr);
        }
    } else {
        grid_sync(a_bar, (unsigned)P);
        trace_mark(tr, 7);
        // shared rows: finished by the owner of their last unit
        for (int t = warp; t < nrow_items; t += kLWarps) {
            const int tb = t / B, b = t - tb * B;
            const int Ir = Ia + (tb >> 4), r = tb & 15;
            const int u0 = Ir * n_units;
            if ((u0 >= L0i && u0 + n_units <= L1i) || owner(u0 + n_units - 1) != c) continue;
            const int i = (tile_row0 + Ir) * kTile + r;
            const float s = warp_row_sum<true>(a_gpart + ((int64_t)b * m_pad + i) * n_units, 1, n_units);
            if (lane == 0) finish(b, i, s);
        }
        if (rht_out) {
            grid_sync(a_bar, (unsigned)P);
            trace_mark(tr, 8);
            rht_out_phase(args, smem, c, P, tr);
        }
    }
    if (tr && threadIdx.x == 0) {
        trace_mark(tr, 11);
        const unsigned long long slot = atomicAdd(g_layer_trace, 1ull);
        if (slot < (unsigned long long)g_layer_trace_cap) {
            unsigned long long* r = g_layer_trace + 1 + (kMarks + 2) * slot;
            r[0] = 5;
            r[1] = blockIdx.x | ((unsigned long long)args.part_smem << 32) | ((unsigned long long)args.stages << 40);
            for (int q = 0; q < kMarks; ++q) r[2 + q] = g_trs[q];
        }
    }
}

// RHT-out, part `part` of `parts`: assemble y~ from ybuf, Sylvester FWHT, write this part's slice of
// y = scale * S_m (H_m^T y~) / sqrt(m) (dense H_b^T mixing of the slice for b > 1).
__device__ __noinline__ void rht_out_phase(const LayerArgs& args, uint8_t* smem, int64_t part, int64_t parts, bool tr) {
    const int64_t m = args.lay.m, m_pad = args.lay.m_pad;
    const int B = args.B;
    const int lenm = (int)m;
    const float os = args.scale * rsqrtf((float)m);
    const int F = B * lenm;
    const int f0 = (int)(part * F / parts), f1 = (int)((part + 1) * F / parts);
    const int Ef = args.mb == 1 ? fwht_fast_E(m, args.ma, kLThreads) : 0;
    if (Ef) {
        float* scr = reinterpret_cast<float*>(smem + args.off_out);
        for (int bt = 0; bt < B; ++bt) {
            if (f1 <= bt * lenm || f0 >= (bt + 1) * lenm) continue;
            auto run = [&](auto EE) {
                constexpr int E = decltype(EE)::value;
                float v[E];
                const int T = lenm / E;
                if ((int)threadIdx.x < T) {
#pragma unroll
                    for (int e = 0; e < E; e += 4) {
                        const float4 q = __ldcg(reinterpret_cast<const float4*>(args.ybuf + bt * m_pad + threadIdx.x * E + e));
                        v[e] = q.x; v[e + 1] = q.y; v[e + 2] = q.z; v[e + 3] = q.w;
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < E; ++e) v[e] = 0.0f;
                }
                trace_mark(tr, 9);
                const int i0 = fwht_fast<E>(v, args.ma, scr);
                trace_mark(tr, 10);
                park_tiles<E>(v, i0, args.ma, scr);
                float* yr = args.y + bt * args.y_stride;
                const int lo = f0 - bt * lenm, hi = f1 - bt * lenm;        // this part's outputs of the row
                for (int tile = (lo > 0 ? lo >> 4 : 0) + threadIdx.x; tile < (lenm >> 4) && 16 * tile < hi;
                     tile += kLThreads) {
                    float o[16];
                    tile_read<E>(scr, tile, o);
                    const uint32_t sb = __ldg(reinterpret_cast<const uint16_t*>(args.sign_m) + tile);
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        o[q] *= os;
                        if ((sb >> q) & 1u) o[q] = -o[q];
                    }
                    if (16 * tile >= lo && 16 * tile + 16 <= hi) {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            *reinterpret_cast<float4*>(yr + 16 * tile + 4 * j) = make_float4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
                    } else {
#pragma unroll
                        for (int q = 0; q < 16; ++q)
                            if (16 * tile + q >= lo && 16 * tile + q < hi) yr[16 * tile + q] = o[q];
                    }
                }
                __syncthreads();
            };
            if (Ef == 4) run(std::integral_constant<int, 4>{});
            else if (Ef == 8) run(std::integral_constant<int, 8>{});
            else run(std::integral_constant<int, 16>{});
        }
        return;
    }
    float* vo = reinterpret_cast<float*>(smem + args.off_out);
    float* ored = reinterpret_cast<float*>(smem + args.off_outred);
    stage_input(vo, lenm, args.ybuf, m_pad, nullptr, B, lenm);
    __syncthreads();
    trace_mark(tr, 9);
    cta_fwht(vo, B * lenm, args.ma);
    trace_mark(tr, 10);
    if (args.mb == 1) {
        for (int f = f0 + threadIdx.x; f < f1; f += kLThreads) {
            const int b = f / lenm, i = f - b * lenm;
            float v = vo[swz(f)] * os;
            if (sgn(args.sign_m, i)) v = -v;
            args.y[b * args.y_stride + i] = v;
        }
    } else {
        const uint8_t* sm_ = args.sign_m;
        float* y = args.y;
        const int64_t ys = args.y_stride;
        dense_mix(vo, lenm, args.mb, args.ma, args.hbt_m, f0, f1, ored, [=](int f, float s) {
            const int b = f / lenm, i = f - b * lenm;
            float v = s * os;
            if (sgn(sm_, i)) v = -v;
            y[b * ys + i] = v;
        });
    }
}

template <int K, int CODE, bool kImm>
cudaError_t launch_layer_t(LayerArgs a, size_t smem, cudaStream_t s) {
    auto kern = layer_kernel<K, CODE, kImm>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kLThreads, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;               // grid barrier needs co-residency
    return launch_coop(kern, dim3((unsigned)num_sms()), dim3(kLThreads), smem, s, a);
}

size_t align128(size_t v) { return (v + 127) & ~(size_t)127; }

// Shared-memory plan; returns 0 when the layer does not fit one CTA per SM.
struct LayerPlan {
    int U, CP, S, max_units, part_smem;
    uint32_t off_lut;
    int64_t T;
    int n_units;
    size_t smem;
    uint32_t off_ring, off_x, off_v, off_red, off_out, off_outred, off_scr;
};

bool plan_layer(const Layout& lay, int code, int64_t B, int64_t tile_rows, bool coop, bool rht_out, int mb,
                LayerPlan* pl, int P_cta = 0) {
    const int P = P_cta > 0 ? P_cta : num_sms();                     // CTAs sharing the layer's tile rows
    const bool hyb = code == QTIP_CODE_HYB;
    const int n_pairs = (int)(lay.n_kc * 4);
    // unit = one cell's tile row (4 tile pairs, 128 columns) for every shape: the association of
    // a row's sum depends on n only, never on m, the row range or the grid
    const int U = 4;
    pl->U = U;
    pl->CP = 4;
    pl->n_units = (n_pairs + U - 1) / U;
    pl->T = tile_rows * pl->n_units;
    pl->max_units = tile_rows >= P ? (int)((tile_rows + P - 1) / P) * pl->n_units   // rows mode (see kernel)
                                   : (int)((pl->T + P - 1) / P);
    const size_t chunk = (size_t)pl->CP * 64 * lay.k;
    const size_t head = 8 * kLWarps * kLMaxStages;
    // unit partials in shared memory whenever the whole plan still fits (else in the workspace)
    const size_t part_bytes = align128((size_t)pl->max_units * kTile * B * 4);
    size_t part = part_bytes;
    pl->part_smem = 1;
    const size_t xs = align128((size_t)B * (lay.n_pad * (hyb ? 2 : 4) + (B > 1 ? (hyb ? 32 : 64) : 0)));   // padded rows
    const size_t vin = align128(((size_t)B * lay.n + 31) / 32 * 32 * 4);
    const size_t vin_pad = align128((size_t)B * lay.n_pad * 4);
    const size_t red = (size_t)kLWarps * kMixChunk * 4;
    const size_t vout = align128(((size_t)B * lay.m + 31) / 32 * 32 * 4);
    const size_t lutb = code == QTIP_CODE_HYB ? (size_t)(512 * 32 * 4) : 0;   // HYB fast path LUT
    auto layout = [&](int S) {                                        // offsets for ring depth S; total bytes
        size_t off = head + part;
        pl->off_lut = (uint32_t)off;
        off += lutb;
        pl->off_ring = (uint32_t)off;
        off += align128((size_t)kLWarps * S * chunk);
        pl->off_x = (uint32_t)off;
        if (coop) {
            pl->off_v = (uint32_t)off;                                // x~ loaded after vin is dead
            off += std::max(xs, vin);
            pl->off_red = (uint32_t)off;
            off += red;
        } else {
            pl->off_v = (uint32_t)off;                                // x~ written in place over vin
            off += std::max(xs, vin_pad);
            pl->off_red = (uint32_t)off;
            pl->off_scr = (uint32_t)off;                              // fast FWHT transpose scratch
            off += align128((size_t)lay.n_pad * 4);
        }
        const size_t endA = off;
        size_t endB = head + part + lutb;                             // RHT-out aliases everything after the LUT
        if (rht_out) {
            pl->off_out = (uint32_t)endB;
            endB += vout;
            pl->off_outred = (uint32_t)endB;
            if (mb > 1) endB += red;
        } else {
            pl->off_out = pl->off_outred = (uint32_t)head;
        }
        return std::max(endA, endB);
    };
    // the deepest ring that still lets a second CTA (the next layer's, under PDL) share the SM,
    // else the deepest that fits one CTA per SM
    int pick = 0;
    for (int pass = 0; pass < 2 && !pick; ++pass) {
        if (pass == 1) {                                              // partials to the workspace instead
            pl->part_smem = 0;
            part = 0;
        }
        for (int S = kLMaxStages; S >= 2 && !pick; --S)
            if (layout(S) <= 113 * 1024) pick = S;
        for (int S = kLMaxStages; S >= 2 && !pick; --S)
            if (layout(S) <= 225 * 1024) pick = S;                     // + static shared memory
    }
    if (!pick) return false;
    pl->S = pick;
    pl->smem = layout(pick);
    return true;
}

}  // namespace

int g_layer_debug = 0;

cudaError_t set_cta_trace_layer(unsigned long long* buf, int cap) {
    cudaError_t e = cudaMemcpyToSymbol(g_layer_trace, &buf, sizeof(buf));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_layer_trace_cap, &cap, sizeof(cap));
    return e;
}

bool layer_supported(const Layout& lay, int code, const CodeArgs& ca, int64_t B, int64_t tile_rows, bool rht_in,
                     bool rht_out) {
    if (B < 1 || B > 4 || lay.k < 2 || lay.k > 4) return false;
    if (code == QTIP_CODE_HYB && ca.Q != 9) return false;   // fast path: 2^9-entry shared-memory LUT
    if (lay.n > (1 << 24) / 4 || lay.m > (1 << 24) / 4 || num_sms() > 256) return false;
    int nb = 1, na = 0, mb = 1, ma = 0;
    if (rht_in && !hadamard_factor(lay.n, &nb, &na)) return false;
    if (rht_out && !hadamard_factor(lay.m, &mb, &ma)) return false;
    LayerPlan pl;
    return plan_layer(lay, code, B, tile_rows, rht_in && nb > 1, rht_out, mb, &pl);
}

size_t layer_workspace_floats(const Layout& lay, int64_t B, int64_t tile_rows) {
    // ybuf [B][m_pad] + gpart [B][m_pad][n_units] (n_units = 2 n_kc)
    (void)tile_rows;
    return (size_t)B * lay.m_pad * (1 + 2 * lay.n_kc);
}

cudaError_t launch_layer(const Layout& lay, int code, const CodeArgs& ca, const void* packed, const uint16_t* lut,
                         const float* x, const uint8_t* sign_n, const uint8_t* sign_m, float scale, float* y,
                         int64_t B, int64_t row_begin, int64_t row_end, bool rht_in, bool rht_out, bool xt_ready,
                         uint32_t* xt_g, int64_t row_words, float* ws_f, unsigned* bar, cudaStream_t s) {
    LayerArgs a{};
    a.packed = (const uint32_t*)packed;
    a.lay = lay;
    a.ca = ca;
    a.lut = (const uint32_t*)lut;
    a.x = x;
    a.sign_n = sign_n;
    a.sign_m = sign_m;
    a.scale = scale;
    a.code_factor = (code == QTIP_CODE_1MAD) ? 5.0f / 739.0f : 1.0f;
    a.y = y;
    a.row_lo = row_begin;
    a.row_hi = row_end;
    a.y_stride = rht_out ? lay.m : row_end - row_begin;
    a.B = (int)B;
    a.rht_in = rht_in;
    a.rht_out = rht_out;
    a.xt_ready = xt_ready;
    a.nb = a.mb = 1;
    a.na = a.ma = 0;
    cudaError_t e = cudaSuccess;
    if (rht_in && !xt_ready) {
        if (!hadamard_factor(lay.n, &a.nb, &a.na)) return cudaErrorInvalidValue;
        if (a.nb > 1) a.hb_n = hadamard_table_device(a.nb, false, &e);
        if (e != cudaSuccess) return e;
    }
    if (rht_out) {
        if (!hadamard_factor(lay.m, &a.mb, &a.ma)) return cudaErrorInvalidValue;
        if (a.mb > 1) a.hbt_m = hadamard_table_device(a.mb, true, &e);
        if (e != cudaSuccess) return e;
    }
    a.coop = rht_in && !xt_ready && a.nb > 1;
    a.xt_g = xt_g;
    a.row_words = row_words;
    a.ybuf = ws_f;
    a.gpart = ws_f + B * lay.m_pad;
    a.bar = bar;
    a.tile_row0 = row_begin / kTile;
    const int64_t tile_rows = (row_end + kTile - 1) / kTile - a.tile_row0;
    LayerPlan pl;
    if (!plan_layer(lay, code, B, tile_rows, a.coop, rht_out, a.mb, &pl)) return cudaErrorInvalidConfiguration;
    a.T = pl.T;
    a.n_units = pl.n_units;
    a.U = pl.U;
    a.CP = pl.CP;
    a.stages = pl.S;
    a.max_units_cta = pl.max_units;
    a.part_smem = pl.part_smem;
    a.off_ring = pl.off_ring;
    a.off_x = pl.off_x;
    a.off_v = pl.off_v;
    a.off_red = pl.off_red;
    a.off_out = pl.off_out;
    a.off_outred = pl.off_outred;
    a.off_scr = pl.off_scr;
    a.off_lut = pl.off_lut;
    a.debug = g_layer_debug;
    a.finishers = (a.mb == 1 && fwht_fast_E(lay.m, a.ma, kLThreads)) ? 1 : std::min(num_sms(), 32);
    const bool imm = code != QTIP_CODE_HYB && ca.a == (code == QTIP_CODE_1MAD ? 34038481u : 89226354u) &&
                     ca.b == (code == QTIP_CODE_1MAD ? 76625530u : 64248484u);
    e = cudaErrorInvalidValue;
#define QTIP_LAYER_CASE(KK, CC)                                                           \
    if (lay.k == KK && code == CC) e = imm ? launch_layer_t<KK, CC, true>(a, pl.smem, s) \
                                           : launch_layer_t<KK, CC, false>(a, pl.smem, s);
    QTIP_LAYER_CASE(2, QTIP_CODE_3INST)
    QTIP_LAYER_CASE(3, QTIP_CODE_3INST)
    QTIP_LAYER_CASE(4, QTIP_CODE_3INST)
    QTIP_LAYER_CASE(2, QTIP_CODE_1MAD)
    QTIP_LAYER_CASE(3, QTIP_CODE_1MAD)
    QTIP_LAYER_CASE(4, QTIP_CODE_1MAD)
    QTIP_LAYER_CASE(2, QTIP_CODE_HYB)
    QTIP_LAYER_CASE(3, QTIP_CODE_HYB)
    QTIP_LAYER_CASE(4, QTIP_CODE_HYB)
#undef QTIP_LAYER_CASE
    count_launch(1);
    return e;
}

bool layer_group_supported(const Layout& lay, int code, const CodeArgs& ca, int64_t B, int G) {
    if (G < 2 || G > kMaxGroup) return false;
    const int64_t tile_rows = (lay.m + kTile - 1) / kTile;
    if (!layer_supported(lay, code, ca, B, tile_rows, false, false)) return false;
    const int P = num_sms();
    if (tile_rows < (P + G - 1) / G) return false;                    // rows mode for every layer
    LayerPlan pl;
    return plan_layer(lay, code, B, tile_rows, false, false, 1, &pl, P / G);
}

cudaError_t launch_layer_group(const Layout& lay, int code, const CodeArgs& ca, int G, const void* const* packed,
                               const uint16_t* const* lut, const float* scale, float* const* y, int64_t B,
                               uint32_t* const* xt_g, int64_t row_words, float* const* ws_f, unsigned* const* bar,
                               cudaStream_t s) {
    if (G < 2 || G > kMaxGroup) return cudaErrorInvalidValue;
    const int P = num_sms();
    const int64_t tile_rows = (lay.m + kTile - 1) / kTile;
    const int Pmin = P / G;
    if (tile_rows < (P + G - 1) / G) return cudaErrorInvalidConfiguration;   // rows mode for every layer
    LayerArgs a{};
    a.packed = (const uint32_t*)packed[0];
    a.lay = lay;
    a.ca = ca;
    a.lut = (const uint32_t*)lut[0];
    a.scale = scale[0];
    a.code_factor = (code == QTIP_CODE_1MAD) ? 5.0f / 739.0f : 1.0f;
    a.y = y[0];
    a.row_lo = 0;
    a.row_hi = lay.m;
    a.y_stride = lay.m;
    a.B = (int)B;
    a.rht_in = a.rht_out = 0;
    a.xt_ready = 1;
    a.nb = a.mb = 1;
    a.coop = 0;
    a.xt_g = xt_g[0];
    a.row_words = row_words;
    a.ybuf = ws_f[0];
    a.gpart = ws_f[0] + B * lay.m_pad;
    a.bar = bar[0];
    a.tile_row0 = 0;
    LayerPlan pl;
    if (!plan_layer(lay, code, B, tile_rows, false, false, 1, &pl, Pmin)) return cudaErrorInvalidConfiguration;
    a.T = pl.T;
    a.n_units = pl.n_units;
    a.U = pl.U;
    a.CP = pl.CP;
    a.stages = pl.S;
    a.max_units_cta = pl.max_units;
    a.part_smem = pl.part_smem;
    a.off_ring = pl.off_ring;
    a.off_x = pl.off_x;
    a.off_v = pl.off_v;
    a.off_red = pl.off_red;
    a.off_out = pl.off_out;
    a.off_outred = pl.off_outred;
    a.off_scr = pl.off_scr;
    a.off_lut = pl.off_lut;
    a.debug = g_layer_debug;
    a.finishers = 1;
    a.G = G;
    for (int g = 0; g <= G; ++g) a.gcta0[g] = (int)((int64_t)g * P / G);
    for (int g = 0; g < G; ++g) {
        a.gpacked[g] = (const uint32_t*)packed[g];
        a.gxt[g] = xt_g[g];
        a.gy[g] = y[g];
        a.gscale[g] = scale[g];
        a.ggpart[g] = ws_f[g] + B * lay.m_pad;
        a.gbar[g] = bar[g];
        a.glut[g] = (const uint32_t*)lut[g];
    }
    const bool imm = code != QTIP_CODE_HYB && ca.a == (code == QTIP_CODE_1MAD ? 34038481u : 89226354u) &&
                     ca.b == (code == QTIP_CODE_1MAD ? 76625530u : 64248484u);
    cudaError_t e = cudaErrorInvalidValue;
#define QTIP_LAYER_CASE(KK, CC)                                                           \
    if (lay.k == KK && code == CC) e = imm ? launch_layer_t<KK, CC, true>(a, pl.smem, s) \
                                           : launch_layer_t<KK, CC, false>(a, pl.smem, s);
    QTIP_LAYER_CASE(2, QTIP_CODE_3INST)
    QTIP_LAYER_CASE(3, QTIP_CODE_3INST)
    QTIP_LAYER_CASE(4, QTIP_CODE_3INST)
    QTIP_LAYER_CASE(2, QTIP_CODE_1MAD)
    QTIP_LAYER_CASE(3, QTIP_CODE_1MAD)
    QTIP_LAYER_CASE(4, QTIP_CODE_1MAD)
    QTIP_LAYER_CASE(2, QTIP_CODE_HYB)
    QTIP_LAYER_CASE(3, QTIP_CODE_HYB)
    QTIP_LAYER_CASE(4, QTIP_CODE_HYB)
#undef QTIP_LAYER_CASE
    count_launch(1);
    return e;
}

}  // namespace qtip
