// k_reduce.cu -- split-K reduction of the per-cell-column partial sums of the GEMV kernels.
//
//   y[b][i - row0] = scale * sum_kc partial[kc][b][i]
// with a fixed association: eight interleaved slices (kc = s mod 8, summed in increasing kc)
// added in slice order.  The order depends only on n, so results are deterministic and a row
// shard reproduces the full call's rows bit for bit.
#include "internal.h"
#include "tc.cuh"

namespace qtip {

constexpr int kRedSlices = 8;

__global__ void __launch_bounds__(256) reduce_kernel(const float* __restrict__ partial, int64_t n_kc, int64_t B,
                                                     int64_t m_pad, int64_t row0, int64_t row1, float scale,
                                                     float* __restrict__ y, int64_t y_stride) {
    __shared__ float part[kRedSlices][33];
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    const int rl = threadIdx.x & 31, sl = threadIdx.x >> 5;
    const int64_t i = row0 + (int64_t)blockIdx.x * 32 + rl;
    const int64_t b = blockIdx.y;
    float s = 0.0f;
    if (i < row1) {
#pragma unroll 4
        for (int64_t kc = sl; kc < n_kc; kc += kRedSlices) s += __ldcg(partial + (kc * B + b) * m_pad + i);
    }
    part[sl][rl] = s;
    __syncthreads();
    if (sl == 0 && i < row1) {
        float t = 0.0f;
#pragma unroll
        for (int q = 0; q < kRedSlices; ++q) t += part[q][rl];
        y[b * y_stride + (i - row0)] = scale * t;
    }
}

cudaError_t launch_reduce(const float* partial, int64_t n_kc, int64_t B, int64_t m_pad, int64_t row0, int64_t row1,
                          float scale, float* y, int64_t y_stride, cudaStream_t s) {
    dim3 grid((unsigned)((row1 - row0 + 31) / 32), (unsigned)B);
    cudaError_t e = launch_pdl(reduce_kernel, grid, dim3(256), 0, s, partial, n_kc, B, m_pad, row0, row1, scale, y,
                               y_stride);
    count_launch(1);
    return e;
}

}  // namespace qtip
