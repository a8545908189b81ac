// k_rht.cu -- random Hadamard transform kernels.
//
// H_n = H_b (x) H_{2^a} (reading R7).  Split 2^a = 2^a1 * 2^a2 and write
// H_n = M_f (x) H_{2^a2} with the "mix" factor M_f = H_b (x) H_{2^a1} of order f = n / 2^a2.
// A CTA owns `rows_per_cta` rows i of M_f: it forms u_i = sum_j M_f[i][j] v_j (v_j the
// j-th length-2^a2 slice of the signed input) and then runs an in-shared-memory fast
// Walsh-Hadamard transform of length 2^a2 on each u_i.  No CTA repeats another's work, and
// every CTA reads the whole (L2-resident) input once.
#include <algorithm>
#include <cmath>

#include "internal.h"

namespace qtip {

constexpr int kRhtThreads = 256;
constexpr int kRhtMaxElems = 4096;   // rows_per_cta * 2^a2 held in shared memory

// out_mode 0: float32; 1: binary16 duplicated into both halves of a 32-bit word (the K-doubled
// UMMA B operand); 2: binary16.
__device__ __forceinline__ void store_out(void* out, int mode, int64_t idx, float v) {
    if (mode == 0) {
        static_cast<float*>(out)[idx] = v;
    } else {
        const uint32_t h = __half_as_ushort(__float2half_rn(v));
        if (mode == 1) static_cast<uint32_t*>(out)[idx] = h | (h << 16);
        else static_cast<uint16_t*>(out)[idx] = (uint16_t)h;
    }
}

__device__ __forceinline__ float sign_of(const uint8_t* __restrict__ s, int64_t i) {
    return ((s[i >> 3] >> (i & 7)) & 1) ? -1.0f : 1.0f;
}

__global__ void __launch_bounds__(kRhtThreads) rht_kernel(RhtPlan plan, const uint8_t* __restrict__ sign,
                                                           const float* __restrict__ in, int64_t in_stride,
                                                           void* __restrict__ out, int64_t out_stride, int inverse,
                                                           float out_scale, int out_mode, int64_t pad_to) {
    __shared__ float buf[kRhtMaxElems];
    __shared__ float part[kRhtThreads];
    const int L2 = 1 << plan.a2;
    const int R = plan.rows_per_cta;
    const int i0 = blockIdx.x * R;
    const int64_t bt = blockIdx.y;
    const float* x = in + bt * in_stride;
    const int a1 = plan.a - plan.a2;
    const int n1 = 1 << a1;
    const int outputs = R * L2;
    const int slices = max(1, kRhtThreads / outputs);          // threads cooperating on one output
    const int tid = threadIdx.x;

    // ---- mix: u[i][c] = sum_j M_f[i][j] * v[j][c]
    for (int o0 = 0; o0 < outputs; o0 += kRhtThreads / slices) {
        const int o = o0 + tid / slices;
        const int sl = tid % slices;
        float acc = 0.0f;
        const int il = o / L2, c = o % L2;
        const int i = i0 + il;
        if (o < outputs && tid / slices < kRhtThreads / slices && i < plan.f) {
            const int ib = i / n1, ia = i % n1;
            for (int j = sl; j < plan.f; j += slices) {
                const int jb = j / n1, ja = j % n1;
                int neg = __popc(ia & ja) & 1;
                if (plan.b > 1) {
                    const int64_t bit = inverse ? ((int64_t)jb * plan.b + ib) : ((int64_t)ib * plan.b + jb);
                    neg ^= (plan.hb[bit >> 5] >> (bit & 31)) & 1;
                }
                const int64_t e = (int64_t)j * L2 + c;
                float v = x[e];
                if (!inverse) v *= sign_of(sign, e);
                acc += neg ? -v : v;
            }
        }
        part[tid] = acc;
        __syncthreads();
        if (sl == 0 && o < outputs && tid / slices < kRhtThreads / slices) {
            float s = 0.0f;
            for (int q = 0; q < slices; ++q) s += part[tid + q];
            buf[o] = s;
        }
        __syncthreads();
    }
    // ---- FWHT of length L2 on each row (butterflies (u+v, u-v) = H_2 on one index bit)
    for (int h = 1; h < L2; h <<= 1) {
        for (int q = tid; q < outputs / 2; q += kRhtThreads) {
            const int row = q / (L2 / 2), k = q % (L2 / 2);
            const int lo = row * L2 + (k / h) * 2 * h + (k % h);
            const float u = buf[lo], v = buf[lo + h];
            buf[lo] = u + v;
            buf[lo + h] = u - v;
        }
        __syncthreads();
    }
    // ---- scale (and signs for the inverse), store
    for (int o = tid; o < outputs; o += kRhtThreads) {
        const int i = i0 + o / L2;
        if (i >= plan.f) continue;
        const int64_t e = (int64_t)i * L2 + (o % L2);
        float v = buf[o] * out_scale;
        if (inverse) v *= sign_of(sign, e);
        store_out(out, out_mode, bt * out_stride + e, v);
    }
    if (blockIdx.x == 0)                                  // zero the padded tail [n, pad_to)
        for (int64_t e = plan.n + tid; e < pad_to; e += kRhtThreads) store_out(out, out_mode, bt * out_stride + e, 0.0f);
}

__global__ void convert_kernel(const float* __restrict__ in, int64_t n, int64_t in_stride, void* __restrict__ out,
                               int64_t out_stride, int out_mode, int64_t pad_to) {
    const int64_t bt = blockIdx.y;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < pad_to; e += (int64_t)gridDim.x * blockDim.x)
        store_out(out, out_mode, bt * out_stride + e, e < n ? in[bt * in_stride + e] : 0.0f);
}

cudaError_t make_rht_plan(int64_t n, RhtPlan* plan) {
    int b, a;
    if (!hadamard_factor(n, &b, &a)) return cudaErrorInvalidValue;
    plan->n = n;
    plan->b = b;
    plan->a = a;
    plan->a2 = a < 10 ? a : 10;
    plan->f = (int)(n >> plan->a2);
    const int L2 = 1 << plan->a2;
    int R = (plan->f + 127) / 128;                 // aim for <= 128 CTAs per batch column
    while (R * L2 > kRhtMaxElems && R > 1) --R;
    if (R * L2 > kRhtMaxElems) return cudaErrorInvalidValue;
    plan->rows_per_cta = R;
    plan->hb = nullptr;
    if (b > 1) {
        cudaError_t err = cudaSuccess;
        plan->hb = hadamard_table_device(b, &err);
        if (!plan->hb) return err == cudaSuccess ? cudaErrorUnknown : err;
    }
    return cudaSuccess;
}

cudaError_t launch_rht(const RhtPlan& plan, int64_t B, const uint8_t* sign, const float* in, int64_t in_stride,
                       void* out, int64_t out_stride, int inverse, float scale, cudaStream_t s, int out_mode,
                       int64_t pad_to) {
    dim3 grid((unsigned)((plan.f + plan.rows_per_cta - 1) / plan.rows_per_cta), (unsigned)B);
    const float out_scale = (float)(scale / std::sqrt((double)plan.n));
    rht_kernel<<<grid, kRhtThreads, 0, s>>>(plan, sign, in, in_stride, out, out_stride, inverse, out_scale, out_mode,
                                            pad_to < plan.n ? plan.n : pad_to);
    count_launch(1);
    return cudaGetLastError();
}

cudaError_t launch_convert(const float* in, int64_t n, int64_t in_stride, int64_t B, void* out, int64_t out_stride,
                           int out_mode, int64_t pad_to, cudaStream_t s) {
    dim3 grid((unsigned)std::min<int64_t>((pad_to + 255) / 256, 1024), (unsigned)B);
    convert_kernel<<<grid, 256, 0, s>>>(in, n, in_stride, out, out_stride, out_mode, pad_to);
    count_launch(1);
    return cudaGetLastError();
}

}  // namespace qtip
