// k_rht.cu -- random Hadamard transform kernels.
//
// H_n = H_b (x) H_{2^a} (reading R7).  With L2 = 2^a2 (a2 = min(a, 8)) write
// H_n = D (x) H_{L2}, D = H_b (x) H_{2^(a-a2)} the dense factor of order f = n / L2,
// D[i][j] = H_b[i_b][j_b] * (-1)^popcount(i_1 & j_1).  Viewing v (n) as V[f][L2]:
//     (H_n v)[i L2 + c] = FWHT_{L2}( sum_j D[i][j] V[j][.] )[c],
// so a CTA owning rows i of D needs every V[j] once and no other CTA's result.
// CTA = 8 warps; a lane owns columns c = lane + 32 e (e < E, L2 = 32 E; for L2 < 32 a warp
// holds 32 / L2 rows side by side) and RA rows of D, and accumulates over its warp's slice of
// j with FFMA against the CTA's rows of D (+-1.0f, built once in shared memory).  The 8 slices are
// added in slice order through shared memory (fixed association: deterministic), then the
// length-L2 Walsh-Hadamard transform runs in registers (bits of e) and warp shuffles (bits of
// the lane) -- no barrier inside the transform.  The input is read straight from global
// memory (L2-resident: the previous kernel just wrote it), coalesced 128 B per row segment.
#include <algorithm>
#include <cmath>
#include <type_traits>

#include "internal.h"
#include "tc.cuh"
#include "trace.cuh"

namespace qtip {

constexpr int kRhtThreads = 256;

// out_mode 6 / 7: the UMMA B layout of the tcgen05 GEMV (k_umma.cu), K-doubled / plain binary16,
// with `stride` = the batch pad BP.
// out_mode 5 = mode 4 with the halves of every pair word swapped (HYB k = 4 fast path, k_layer.cu).
// out_mode 0: float32; 1: binary16 duplicated into both halves of a 32-bit word (the K-doubled
// UMMA B operand); 2: binary16; 3 / 4: modes 1 / 2 permuted into mma.sync B-fragment order
// within each 16-column tile (k_gemv_mma.cu): mode 3 puts columns (2t, 2t+8, 2t+1, 2t+9) at
// words 4t .. 4t+3, mode 4 puts the pairs (t, t+4) at words 2t, 2t+1.  `row` is the element
// offset of the batch row, e the column.
__device__ __forceinline__ void store_out(void* out, int mode, int64_t bt, int64_t stride, int64_t e, float v) {
    const int64_t row = bt * stride;
    if (mode == 0) {
        static_cast<float*>(out)[row + e] = v;
        return;
    }
    const uint32_t h = __half_as_ushort(__float2half_rn(v));
    const int64_t tile = e >> 4;
    const int c = (int)(e & 15);
    if (mode == 1) {
        static_cast<uint32_t*>(out)[row + e] = h | (h << 16);
    } else if (mode == 2) {
        static_cast<uint16_t*>(out)[row + e] = (uint16_t)h;
    } else if (mode == 6) {
        // UMMA B operand, K-doubled (k_umma.cu): 16-byte K chunks of 4 columns, batch rows interleaved
        // per chunk (stride = BP rows)
        static_cast<uint32_t*>(out)[(e >> 2) * 4 * stride + 4 * bt + (e & 3)] = h | (h << 16);
    } else if (mode == 7) {
        // UMMA B operand, plain binary16 (HYB): 16-byte K chunks of 8 columns, batch rows interleaved
        static_cast<uint16_t*>(out)[(e >> 3) * 8 * stride + 8 * bt + (e & 7)] = (uint16_t)h;
    } else if (mode == 3) {
        const int t = (c & 7) >> 1, q = ((c & 1) << 1) | (c >> 3);
        static_cast<uint32_t*>(out)[row + tile * 16 + 4 * t + q] = h | (h << 16);
    } else {
        const int j = c >> 1;                                  // column pair
        const int64_t w = tile * 8 + 2 * (j & 3) + (j >> 2);
        // mode 5 (HYB fast path): the two halves of each pair word swapped (LUT words (c0 << 16) | c1)
        static_cast<uint16_t*>(out)[row + 2 * w + ((c & 1) ^ (mode == 5 ? 1 : 0))] = (uint16_t)h;
    }
}

__device__ __forceinline__ uint32_t sign_bit(const uint8_t* __restrict__ s, int64_t i) {
    return (s[i >> 3] >> (i & 7)) & 1u;
}

constexpr int kRhtWarps = kRhtThreads / 32;

__device__ unsigned long long* g_rht_trace = nullptr;
__device__ int g_rht_trace_cap = 0;

// Per-transform pointers of a (grouped) launch: transform z = blockIdx.z uses entry z.
struct RhtIO {
    const uint8_t* sign[kMaxGroup];
    const float* in[kMaxGroup];
    void* out[kMaxGroup];
    float out_scale[kMaxGroup];
    int* zero[kMaxGroup];                                    // cleared after the PDL wait (the GEMV's counters)
    int zero_n;
    const uint8_t* pf[kMaxGroup];                            // L2 prefetch of the next GEMV's weights (or null)
    uint64_t pf_bytes[kMaxGroup];
};

// Pending L2 prefetch for the next RHT launch on this host thread (rht_set_prefetch): the RHT-in
// kernel of a layer prefetches that layer's packed weights into L2 before its PDL wait -- the
// weights are static, so the prefetch overlaps the previous kernels, and the GEMV that follows
// starts on L2 hits instead of HBM latency.
static thread_local RhtIO t_pf{};
void rht_set_prefetch(int G, const void* const* ptr, const uint64_t* bytes) {
    for (int g = 0; g < kMaxGroup; ++g) {
        t_pf.pf[g] = g < G ? (const uint8_t*)ptr[g] : nullptr;
        t_pf.pf_bytes[g] = g < G ? bytes[g] : 0;
    }
}

// the batched plans (E = 1, RA >= 8: n = 11008, B = 16 -> 352 CTAs) fit one wave at 3 CTAs per SM
template <int E, int RA>
__global__ void __launch_bounds__(kRhtThreads, (E == 1 && RA >= 8) ? 3 : 1) rht_kernel(RhtPlan plan, const __grid_constant__ RhtIO io,
                                                           int64_t in_stride, int64_t out_stride, int inverse,
                                                           int out_mode, int64_t pad_to,
                                                           int* __restrict__ zero_ptr, int zero_n) {
    extern __shared__ __align__(16) float sm[];
    const int z = blockIdx.z;
    const uint8_t* __restrict__ sign = io.sign[z];
    const float* __restrict__ in = io.in[z];
    void* __restrict__ out = io.out[z];
    const float out_scale = io.out_scale[z];
    const int L2 = 1 << plan.a2;
    const int CL = L2 < 32 ? L2 : 32;                        // lanes per row
    const int rpw = 32 / CL;                                 // rows side by side in a warp
    const int R = plan.rows_per_cta;                         // = RA * rpw
    const int f = plan.f;
    float* Dsm = sm;                                         // [f][R] +-1.0f (row r0 + rl of D, column j)
    float* red = sm + ((f * R + 3) & ~3);                    // [8][R][L2] slice partial sums
    uint32_t* ssm = reinterpret_cast<uint32_t*>(red + kRhtWarps * R * L2);   // forward: sign bits, n / 32 words
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int c = lane & (CL - 1), ro = lane / CL;
    const int r0 = blockIdx.x * R;
    const int64_t bt = blockIdx.y;
    const int a1 = plan.a - plan.a2, m1 = (1 << a1) - 1;
    __shared__ unsigned long long trace_ts[4];
    CtaTrace trace{trace_ts};
    trace.entry(g_rht_trace);

    // L2 prefetch of the next GEMV's weights (static data: before the PDL wait), one slice per CTA
    if (tid == 0 && io.pf[z] != nullptr) {
        const uint64_t ncta = (uint64_t)gridDim.x * gridDim.y, cid = (uint64_t)blockIdx.y * gridDim.x + blockIdx.x;
        const uint64_t per = ((io.pf_bytes[z] + ncta - 1) / ncta + 15) & ~15ull;
        const uint64_t lo = cid * per, hi = lo + per < io.pf_bytes[z] ? lo + per : io.pf_bytes[z];
        for (uint64_t o = lo; o < hi; o += 65536) ptx::bulk_prefetch_l2(io.pf[z] + o, (uint32_t)(hi - o < 65536 ? hi - o : 65536));
    }
    // D rows of this CTA (static tables only: overlaps the previous kernel under PDL)
    {
        const uint32_t* hb = inverse ? plan.hbt : plan.hb;
        const int wpr = (plan.b + 31) >> 5;
        const int lgR = __ffs(R) - 1;                        // R = RA x rows per warp: a power of two
        for (int e = tid; e < f * R; e += kRhtThreads) {
            const int j = e >> lgR, rl = e & (R - 1), r = r0 + rl;   // (a runtime division here was
                                                                     // 29 % of the batched kernel's instructions)
            float d = 0.0f;
            if (r < f) {
                const int ib = r >> a1, jb = j >> a1;
                uint32_t neg = __popc((r & m1) & (j & m1)) & 1u;
                if (plan.b > 1) neg ^= (__ldg(hb + ib * wpr + (jb >> 5)) >> (jb & 31)) & 1u;
                d = neg ? -1.0f : 1.0f;
            }
            Dsm[e] = d;
        }
    }
    const bool sign_words = !inverse && CL == 32 && (reinterpret_cast<uintptr_t>(sign) & 3u) == 0;
    if (sign_words)                                          // n % 32 == 0 here
        for (int w = tid; w < (int)(plan.n >> 5); w += kRhtThreads) ssm[w] = __ldg(reinterpret_cast<const uint32_t*>(sign) + w);
    ptx::pdl_wait();                                         // the input may be the previous kernel's output
    ptx::pdl_launch_dependents();
    trace.waited(g_rht_trace);
    if (blockIdx.x == 0 && blockIdx.y == 0 && z == 0)
        for (int i = tid; i < zero_n; i += kRhtThreads) zero_ptr[i] = 0;
    if (blockIdx.x == 0 && blockIdx.y == 0 && io.zero[z])
        for (int i = tid; i < io.zero_n; i += kRhtThreads) io.zero[z][i] = 0;
    __syncthreads();

    // slice sums: acc[q][e] = sum_{j in slice} D[r0 + ro RA + q][j] V[j][c + 32 e]
    float acc[RA][E];
#pragma unroll
    for (int q = 0; q < RA; ++q)
#pragma unroll
        for (int e = 0; e < E; ++e) acc[q][e] = 0.0f;
    const float* x = in + bt * in_stride;
    const int j_lo = f * warp / kRhtWarps, j_hi = f * (warp + 1) / kRhtWarps;
    // loads of U rows are issued together before their FMAs (the latency is L2's, ~U x fewer round trips)
    auto slice = [&](auto kind) {
        constexpr int K = decltype(kind)::value;             // 0 plain, 1 sign words, 2 sign bytes
        // rows whose loads are issued together (f = 128, n = 4096: one round per warp)
        constexpr int U = E >= 4 ? 2 : 16;
        const float* xp = x + (int64_t)j_lo * L2 + c;
        int j = j_lo;
        auto step = [&](const float (&v)[E], int jj) {
            const float* d = Dsm + jj * R + ro * RA;
            if constexpr (RA % 4 == 0) {
                // four rows of D per (broadcast) LDS.128: with one LDS per FFMA the shared-memory pipe,
                // not the FMAs, bound the batched transforms (n = 11008, B = 16: RA = 16)
#pragma unroll
                for (int q4 = 0; q4 < RA; q4 += 4) {
                    const float4 d4 = *reinterpret_cast<const float4*>(d + q4);
                    const float dq[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq)
#pragma unroll
                        for (int e = 0; e < E; ++e) acc[q4 + qq][e] = fmaf(dq[qq], v[e], acc[q4 + qq][e]);
                }
            } else {
#pragma unroll
                for (int q = 0; q < RA; ++q) {
                    const float dq = d[q];
#pragma unroll
                    for (int e = 0; e < E; ++e) acc[q][e] = fmaf(dq, v[e], acc[q][e]);
                }
            }
        };
        auto load = [&](float (&v)[E], int jj) {
            const float* p = xp + (int64_t)(jj - j_lo) * L2;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                v[e] = __ldg(p + 32 * e);
                if constexpr (K == 1) {
                    const uint32_t w = ssm[((jj * L2) >> 5) + e];
                    v[e] = __int_as_float(__float_as_int(v[e]) ^ ((w << (31 - lane)) & 0x80000000u));
                } else if constexpr (K == 2) {
                    if (sign_bit(sign, (int64_t)jj * L2 + c + 32 * e)) v[e] = -v[e];
                }
            }
        };
        for (; j + U <= j_hi; j += U) {
            float v[U][E];
#pragma unroll
            for (int u = 0; u < U; ++u) load(v[u], j + u);
#pragma unroll
            for (int u = 0; u < U; ++u) step(v[u], j + u);
        }
        if (j < j_hi) {                                      // the tail: one predicated round, not one
            const int rem = j_hi - j;                        // L2 round trip per row (n = 11008: 43 rows
            float v[U][E];                                   // per warp = 2 rounds + 11 singles before)
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (u < rem) load(v[u], j + u);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (u < rem) step(v[u], j + u);
        }
    };
    if (inverse) slice(std::integral_constant<int, 0>{});
    else if (sign_words) slice(std::integral_constant<int, 1>{});
    else slice(std::integral_constant<int, 2>{});
#pragma unroll
    for (int q = 0; q < RA; ++q)
#pragma unroll
        for (int e = 0; e < E; ++e) red[(warp * R + ro * RA + q) * L2 + c + 32 * e] = acc[q][e];
    __syncthreads();

    // rows ro RA + q, q = warp, warp + 8, ...: sum the 8 slices in order, FWHT, store
    for (int q = warp; q < RA; q += kRhtWarps) {
        const int rl = ro * RA + q, r = r0 + rl;
        float u[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            float t = 0.0f;
#pragma unroll
            for (int w = 0; w < kRhtWarps; ++w) t += red[(w * R + rl) * L2 + c + 32 * e];
            u[e] = t;
        }
        // butterflies on the column bits held by the lane (distance < CL): shuffles
        for (int h = 1; h < CL; h <<= 1) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const float o = __shfl_xor_sync(0xffffffffu, u[e], h);
                u[e] = (c & h) ? (o - u[e]) : (u[e] + o);
            }
        }
        // butterflies on the bits of e (distance 32, 64, ...): in registers
#pragma unroll
        for (int h = 1; h < E; h <<= 1) {
#pragma unroll
            for (int e = 0; e < E; ++e)
                if (!(e & h)) {
                    const float lo = u[e], hi = u[e | h];
                    u[e] = lo + hi;
                    u[e | h] = lo - hi;
                }
        }
        if (r < f) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int64_t idx = (int64_t)r * L2 + c + 32 * e;
                float o = u[e] * out_scale;
                if (inverse && sign_bit(sign, idx)) o = -o;
                store_out(out, out_mode, bt, out_stride, idx, o);
            }
        }
    }
    if (blockIdx.x == 0)                                     // zero the padded tail [n, pad_to)
        for (int64_t e = plan.n + tid; e < pad_to; e += kRhtThreads) store_out(out, out_mode, bt, out_stride, e, 0.0f);
    trace.exit(g_rht_trace, inverse ? 2 : 1, g_rht_trace_cap);
}

__global__ void convert_kernel(const float* __restrict__ in, int64_t n, int64_t in_stride, void* __restrict__ out,
                               int64_t out_stride, int out_mode, int64_t pad_to, int* __restrict__ zero_ptr, int zero_n) {
    const int64_t bt = blockIdx.y;
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    if (blockIdx.x == 0 && blockIdx.y == 0)
        for (int i = threadIdx.x; i < zero_n; i += blockDim.x) zero_ptr[i] = 0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < pad_to; e += (int64_t)gridDim.x * blockDim.x)
        store_out(out, out_mode, bt, out_stride, e, e < n ? in[bt * in_stride + e] : 0.0f);
}

constexpr int64_t kRhtMaxN = 48 * 1024;

cudaError_t make_rht_plan(int64_t n, RhtPlan* plan, int min_ctas, int64_t B) {
    int b, a;
    if (!hadamard_factor(n, &b, &a)) return cudaErrorInvalidValue;
    if (n > kRhtMaxN) return cudaErrorInvalidValue;
    plan->n = n;
    plan->b = b;
    plan->a = a;
    // a2 = 5 (one column per lane, the whole transform tail in 5 shuffles, 4 rows per lane) while
    // the dense factor stays small; longer Walsh-Hadamard factors otherwise (less L2 re-reading)
    plan->a2 = a < 8 ? a : 8;
    if (a >= 5 && (n >> 5) <= 512) plan->a2 = 5;
    const int L2 = 1 << plan->a2;
    plan->f = (int)(n >> plan->a2);
    plan->E = L2 >= 32 ? L2 / 32 : 1;
    const int rpw = L2 >= 32 ? 1 : 32 / L2;
    // rows per lane: amortise the D loads, but keep at least ~one CTA per SM when f allows.  Every
    // CTA reads its whole input vector from L2, so the L2 traffic is (CTAs per vector) x B x 4n:
    // with a batch the CTAs take more rows of D (up to 16) while B x (CTAs per vector) >= min_ctas
    // (n = 11008, B = 16: 172 -> 22 CTAs per vector, 121 -> 15 MB of L2 reads)
    int RA = 1;
    if (plan->E <= 2 || B > 1) {
        RA = B <= 1 ? 4 : (plan->E == 1 ? 16 : plan->E == 2 ? 8 : 4);
        while (RA > 1 && B * ((plan->f + RA * rpw - 1) / (RA * rpw)) < min_ctas) RA /= 2;
    }
    plan->RA = RA;
    plan->rows_per_cta = RA * rpw;
    plan->hb = plan->hbt = nullptr;
    if (b > 1) {
        cudaError_t err = cudaSuccess;
        plan->hb = hadamard_table_device(b, false, &err);
        if (!plan->hb) return err == cudaSuccess ? cudaErrorUnknown : err;
        plan->hbt = hadamard_table_device(b, true, &err);
        if (!plan->hbt) return err == cudaSuccess ? cudaErrorUnknown : err;
    }
    return cudaSuccess;
}

template <int E, int RA>
static cudaError_t launch_rht_t(const RhtPlan& plan, int G, int64_t B, const RhtIO& io, int64_t in_stride,
                                int64_t out_stride, int inverse, cudaStream_t s, int out_mode, int64_t pad,
                                int* zero_ptr, int zero_n) {
    const int L2 = 1 << plan.a2;
    const size_t smem = sizeof(float) * ((size_t)((plan.f * plan.rows_per_cta + 3) & ~3) +
                                         (size_t)kRhtWarps * plan.rows_per_cta * L2 + (size_t)(plan.n >> 5));
    auto kern = rht_kernel<E, RA>;
    // the attribute is per device: set it on every launch (cheap; graphs replay without it)
    cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (ea != cudaSuccess) return ea;
    dim3 grid((unsigned)((plan.f + plan.rows_per_cta - 1) / plan.rows_per_cta), (unsigned)B, (unsigned)G);
    return launch_pdl(kern, grid, dim3(kRhtThreads), smem, s, plan, io, in_stride, out_stride, inverse, out_mode, pad,
                      zero_ptr, zero_n);
}

static cudaError_t launch_rht_io(const RhtPlan& plan, int G, int64_t B, const RhtIO& io_in, int64_t in_stride,
                                 int64_t out_stride, int inverse, cudaStream_t s, int out_mode, int64_t pad_to,
                                 int* zero_ptr, int zero_n) {
    RhtIO io = io_in;
    for (int g = 0; g < kMaxGroup; ++g) {                   // take (and clear) the pending prefetch
        io.pf[g] = t_pf.pf[g];
        io.pf_bytes[g] = t_pf.pf_bytes[g];
        t_pf.pf[g] = nullptr;
        t_pf.pf_bytes[g] = 0;
    }
    const int64_t pad = pad_to < plan.n ? plan.n : pad_to;
    cudaError_t e = cudaErrorInvalidValue;
#define QTIP_RHT_CASE(EE, RR) \
    if (plan.E == EE && plan.RA == RR) e = launch_rht_t<EE, RR>(plan, G, B, io, in_stride, out_stride, inverse, s, out_mode, pad, zero_ptr, zero_n);
    QTIP_RHT_CASE(1, 1) QTIP_RHT_CASE(1, 2) QTIP_RHT_CASE(1, 4) QTIP_RHT_CASE(1, 8) QTIP_RHT_CASE(1, 16)
    QTIP_RHT_CASE(2, 1) QTIP_RHT_CASE(2, 2) QTIP_RHT_CASE(2, 4) QTIP_RHT_CASE(2, 8) QTIP_RHT_CASE(4, 1)
    QTIP_RHT_CASE(4, 2) QTIP_RHT_CASE(4, 4) QTIP_RHT_CASE(8, 1) QTIP_RHT_CASE(8, 2) QTIP_RHT_CASE(8, 4)
#undef QTIP_RHT_CASE
    count_launch(1);
    return e;
}

cudaError_t launch_rht(const RhtPlan& plan, int64_t B, const uint8_t* sign, const float* in, int64_t in_stride,
                       void* out, int64_t out_stride, int inverse, float scale, cudaStream_t s, int out_mode,
                       int64_t pad_to, int* zero_ptr, int zero_n) {
    RhtIO io{};
    io.sign[0] = sign;
    io.in[0] = in;
    io.out[0] = out;
    io.out_scale[0] = (float)(scale / std::sqrt((double)plan.n));
    return launch_rht_io(plan, 1, B, io, in_stride, out_stride, inverse, s, out_mode, pad_to, zero_ptr, zero_n);
}

cudaError_t launch_rht_group(const RhtPlan& plan, int G, int64_t B, const uint8_t* const* sign, const float* const* in,
                             int64_t in_stride, void* const* out, int64_t out_stride, int inverse, const float* scale,
                             cudaStream_t s, int out_mode, int64_t pad_to, int* const* zero, int zero_n) {
    if (G < 1 || G > kMaxGroup) return cudaErrorInvalidValue;
    RhtIO io{};
    io.zero_n = zero ? zero_n : 0;
    for (int g = 0; g < G; ++g) {
        io.zero[g] = zero ? zero[g] : nullptr;
        io.sign[g] = sign[g];
        io.in[g] = in[g];
        io.out[g] = out[g];
        io.out_scale[g] = (float)(scale[g] / std::sqrt((double)plan.n));
    }
    return launch_rht_io(plan, G, B, io, in_stride, out_stride, inverse, s, out_mode, pad_to, nullptr, 0);
}

cudaError_t launch_convert(const float* in, int64_t n, int64_t in_stride, int64_t B, void* out, int64_t out_stride,
                           int out_mode, int64_t pad_to, cudaStream_t s, int* zero_ptr, int zero_n) {
    dim3 grid((unsigned)std::min<int64_t>((pad_to + 255) / 256, 1024), (unsigned)B);
    cudaError_t e = launch_pdl(convert_kernel, grid, dim3(256), 0, s, in, n, in_stride, out, out_stride, out_mode, pad_to,
                               zero_ptr, zero_n);
    count_launch(1);
    return e;
}

cudaError_t set_cta_trace_rht(unsigned long long* buf, int cap) {
    cudaError_t e = cudaMemcpyToSymbol(g_rht_trace, &buf, sizeof(buf));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_rht_trace_cap, &cap, sizeof(cap));
    return e;
}

}  // namespace qtip
