// k_rht.cu -- random Hadamard transform kernels.
//
// H_n = H_b (x) H_{2^a} (reading R7).  Split 2^a = 2^a1 * 2^a2 (2^a2 <= 256) and write
// H_n = M_f (x) H_{2^a2} with the "mix" factor M_f = H_b (x) H_{2^a1} of order f = n / 2^a2,
// M_f[i][j] = H_b[i_b][j_b] * (-1)^popcount(i_a1 & j_a1).
// One CTA of 256 threads owns R = 256 / 2^a2 rows i of M_f (one output per thread):
//   1. stage the whole signed input (n floats, coalesced float4) in shared memory,
//   2. u_i[c] = sum_j M_f[i][j] v_j[c] from shared memory (sign bits of its H_b row in smem),
//   3. fast Walsh-Hadamard transform of length 2^a2 across the threads: butterflies with
//      partner distance < 32 via warp shuffles, the rest through shared memory,
//   4. scale (and the output signs for the inverse), coalesced store.
// No CTA repeats another's arithmetic; every CTA reads the (L2-resident) input once.
#include <algorithm>
#include <cmath>

#include "internal.h"
#include "tc.cuh"

namespace qtip {

constexpr int kRhtThreads = 256;

// out_mode 0: float32; 1: binary16 duplicated into both halves of a 32-bit word (the K-doubled
// UMMA B operand); 2: binary16; 3 / 4: modes 1 / 2 permuted into mma.sync B-fragment order
// within each 16-column tile (k_gemv_mma.cu): mode 3 puts columns (2t, 2t+8, 2t+1, 2t+9) at
// words 4t .. 4t+3, mode 4 puts the pairs (t, t+4) at words 2t, 2t+1.  `row` is the element
// offset of the batch row, e the column.
__device__ __forceinline__ void store_out(void* out, int mode, int64_t row, int64_t e, float v) {
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
    } else if (mode == 3) {
        const int t = (c & 7) >> 1, q = ((c & 1) << 1) | (c >> 3);
        static_cast<uint32_t*>(out)[row + tile * 16 + 4 * t + q] = h | (h << 16);
    } else {
        const int j = c >> 1;                                  // column pair
        const int64_t w = tile * 8 + 2 * (j & 3) + (j >> 2);
        static_cast<uint16_t*>(out)[row + 2 * w + (c & 1)] = (uint16_t)h;
    }
}

__device__ __forceinline__ uint32_t sign_bit(const uint8_t* __restrict__ s, int64_t i) {
    return (s[i >> 3] >> (i & 7)) & 1u;
}

__global__ void __launch_bounds__(kRhtThreads) rht_kernel(RhtPlan plan, const uint8_t* __restrict__ sign,
                                                           const float* __restrict__ in, int64_t in_stride,
                                                           void* __restrict__ out, int64_t out_stride, int inverse,
                                                           float out_scale, int out_mode, int64_t pad_to) {
    extern __shared__ __align__(16) float xs[];             // [n] staged input, then [256] FWHT exchange
    __shared__ uint32_t hrow[64][32];                        // H_b (or H_b^T) rows of this CTA's rows, bits
    const int L2 = 1 << plan.a2;
    const int R = plan.rows_per_cta;                         // rows of M_f per CTA
    const int RL = R * L2;                                   // outputs per CTA
    const int S = kRhtThreads / RL;                          // threads (j-slices) per output
    const int tid = threadIdx.x;
    const int sl = tid / RL, il = (tid % RL) >> plan.a2, c = tid & (L2 - 1);
    const int i = blockIdx.x * R + il;                       // row of M_f
    const int64_t bt = blockIdx.y;
    const int n1 = 1 << (plan.a - plan.a2);
    const int n = (int)plan.n;
    const float* x = in + bt * in_stride;

    ptx::pdl_wait();                                         // the input may be the previous kernel's output
    ptx::pdl_launch_dependents();

    // 1. stage v = (S .) x into shared memory (loads batched 8 deep to overlap their latency)
    for (int e0 = 4 * tid; e0 < n; e0 += 4 * kRhtThreads * 8) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = e0 + 4 * kRhtThreads * u;
            if (e < n) v[u] = __ldg(reinterpret_cast<const float4*>(x + e));
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = e0 + 4 * kRhtThreads * u;
            if (e < n) {
                if (!inverse) {
                    const uint32_t sb = (sign[e >> 3] >> (e & 7)) & 0xFu;   // e % 4 == 0: four bits of one byte
                    v[u].x = (sb & 1u) ? -v[u].x : v[u].x;
                    v[u].y = (sb & 2u) ? -v[u].y : v[u].y;
                    v[u].z = (sb & 4u) ? -v[u].z : v[u].z;
                    v[u].w = (sb & 8u) ? -v[u].w : v[u].w;
                }
                *reinterpret_cast<float4*>(xs + e) = v[u];
            }
        }
    }
    if (plan.b > 1) {
        const int wpr = (plan.b + 31) >> 5;
        for (int e = tid; e < R * wpr; e += kRhtThreads) {
            const int rl = e / wpr, w = e % wpr;
            const int ib = min(blockIdx.x * R + rl, plan.f - 1) / n1;
            hrow[rl][w] = (inverse ? plan.hbt : plan.hb)[ib * wpr + w];
        }
    }
    __syncthreads();

    // 2. mix: u = sum_j M_f[i][j] v[j][c], the j-sum split over S slices (j_b = sl mod S)
    //    that are added in slice order (a fixed association: deterministic)
    float acc = 0.0f;
    if (i < plan.f) {
        const int ia = i & (n1 - 1);
        for (int jb = sl; jb < plan.b; jb += S) {
            const uint32_t sb = (plan.b > 1) ? ((hrow[il][jb >> 5] >> (jb & 31)) & 1u) : 0u;
#pragma unroll 4
            for (int ja = 0; ja < n1; ++ja) {
                const uint32_t neg = sb ^ (__popc(ia & ja) & 1u);
                const float v = xs[(jb * n1 + ja) * L2 + c];
                acc += __int_as_float(__float_as_int(v) ^ (neg << 31));
            }
        }
    }
    __syncthreads();                                         // xs is reused below
    if (S > 1) {
        xs[tid] = acc;
        __syncthreads();
        if (tid < RL) {
            acc = 0.0f;
            for (int q = 0; q < S; ++q) acc += xs[q * RL + tid];
        }
        __syncthreads();
    }
    // 3. FWHT of length L2 along c (threads < R L2 hold the values; all threads run the loop so the
    //    shuffles and barriers stay uniform): lower index of a pair gets u + v, upper gets u - v
    for (int h = 1; h < L2; h <<= 1) {
        float other;
        if (h < 32) {
            other = __shfl_xor_sync(0xffffffffu, acc, h);
        } else {
            xs[tid] = acc;
            __syncthreads();
            other = xs[tid ^ h];
            __syncthreads();
        }
        acc = (c & h) ? (other - acc) : (acc + other);
    }
    // 4. scale (and signs for the inverse), store
    if (sl == 0 && i < plan.f) {
        const int64_t e = (int64_t)i * L2 + c;
        float v = acc * out_scale;
        if (inverse && sign_bit(sign, e)) v = -v;
        store_out(out, out_mode, bt * out_stride, e, v);
    }
    if (blockIdx.x == 0)                                     // zero the padded tail [n, pad_to)
        for (int64_t e = plan.n + tid; e < pad_to; e += kRhtThreads) store_out(out, out_mode, bt * out_stride, e, 0.0f);
}

__global__ void convert_kernel(const float* __restrict__ in, int64_t n, int64_t in_stride, void* __restrict__ out,
                               int64_t out_stride, int out_mode, int64_t pad_to) {
    const int64_t bt = blockIdx.y;
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < pad_to; e += (int64_t)gridDim.x * blockDim.x)
        store_out(out, out_mode, bt * out_stride, e, e < n ? in[bt * in_stride + e] : 0.0f);
}

constexpr int64_t kRhtMaxN = 48 * 1024;                      // staged input <= 192 KB of shared memory

cudaError_t make_rht_plan(int64_t n, RhtPlan* plan) {
    int b, a;
    if (!hadamard_factor(n, &b, &a)) return cudaErrorInvalidValue;
    if (n > kRhtMaxN || n % 4) return cudaErrorInvalidValue;
    plan->n = n;
    plan->b = b;
    plan->a = a;
    plan->a2 = a < 8 ? a : 8;
    plan->f = (int)(n >> plan->a2);
    // at least one warp of outputs per CTA, at most ~2 waves of CTAs; the rest of the 256
    // threads split each output's j-sum
    const int L2 = 1 << plan->a2;
    int R = std::max(1, 32 / L2);
    while ((plan->f + R - 1) / R > 296 && R * L2 < kRhtThreads) R *= 2;
    plan->rows_per_cta = R;
    if (R * L2 > kRhtThreads || R > 64 || kRhtThreads % (R * L2)) return cudaErrorInvalidValue;
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

cudaError_t launch_rht(const RhtPlan& plan, int64_t B, const uint8_t* sign, const float* in, int64_t in_stride,
                       void* out, int64_t out_stride, int inverse, float scale, cudaStream_t s, int out_mode,
                       int64_t pad_to) {
    dim3 grid((unsigned)((plan.f + plan.rows_per_cta - 1) / plan.rows_per_cta), (unsigned)B);
    const float out_scale = (float)(scale / std::sqrt((double)plan.n));
    const int64_t pad = pad_to < plan.n ? plan.n : pad_to;
    const size_t smem = (size_t)std::max<int64_t>(plan.n, kRhtThreads) * sizeof(float);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(rht_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kRhtMaxN * sizeof(float)));
        attr_set = true;
    }
    cudaError_t e = launch_pdl(rht_kernel, grid, dim3(kRhtThreads), smem, s, plan, sign, in, in_stride, out,
                               out_stride, inverse, out_scale, out_mode, pad);
    count_launch(1);
    return e;
}

cudaError_t launch_convert(const float* in, int64_t n, int64_t in_stride, int64_t B, void* out, int64_t out_stride,
                           int out_mode, int64_t pad_to, cudaStream_t s) {
    dim3 grid((unsigned)std::min<int64_t>((pad_to + 255) / 256, 1024), (unsigned)B);
    cudaError_t e = launch_pdl(convert_kernel, grid, dim3(256), 0, s, in, n, in_stride, out, out_stride, out_mode, pad_to);
    count_launch(1);
    return e;
}

}  // namespace qtip
