// k_gemv_simple.cu -- reference CUDA-core fused decode + GEMV (impl 1) and the split-K reduce.
//
// One CTA per (row block of 128, K-chunk of 128 columns), one thread per output row; the
// thread decodes its row of each tile (decode.cuh, bit-identical to qtip_decode) and
// accumulates fp16-exact weights times fp32 x~ with FFMA.  Partial sums per K-chunk go to
// the workspace and are summed in fixed chunk order (deterministic, shard-invariant).
#include "decode.cuh"
#include "internal.h"

namespace qtip {

constexpr int kSimpleNB = 8;   // batch columns per pass

template <int K, int V, int CODE>
__global__ void __launch_bounds__(128) gemv_simple_kernel(const uint32_t* __restrict__ packed, Layout lay, CodeArgs ca,
                                                          const uint16_t* __restrict__ lut,
                                                          const float* __restrict__ xt, int B, int64_t rb0,
                                                          float* __restrict__ partial) {
    extern __shared__ float xs[];                 // [B][128] slice of x~ for this K-chunk
    const int KC = blockIdx.x;
    const int64_t RB = rb0 + blockIdx.y;
    const int t = threadIdx.x, I = t >> 4, r = t & 15;
    for (int e = t; e < B * kCellCols; e += 128) {
        const int b = e / kCellCols, c = e % kCellCols;
        const int64_t col = (int64_t)KC * kCellCols + c;
        xs[e] = col < lay.n ? xt[(int64_t)b * lay.n_pad + col] : 0.0f;
    }
    __syncthreads();
    const uint32_t* cell = packed + (RB * lay.n_kc + KC) * lay.cell_words;
    const int64_t row = RB * kCellRows + t;
    for (int b0 = 0; b0 < B; b0 += kSimpleNB) {
        float acc[kSimpleNB];
#pragma unroll
        for (int i = 0; i < kSimpleNB; ++i) acc[i] = 0.0f;
#pragma unroll 1
        for (int J = 0; J < kCellTileCols; ++J) {
            uint16_t v[16];
            // decode (shared with qtip_decode through decode.cuh)
            constexpr int TW = 8 * K;
            if constexpr (K == 2 && V == 1) {
                const uint32_t A = cell[cell_word_index(I, J, r, TW)];
                const uint32_t Bw = cell[cell_word_index(I, J, (r + 1) & 15, TW)];
                uint32_t x[16];
                windows_k2v1(A, Bw, x);
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    v[q] = (CODE == QTIP_CODE_3INST) ? __half_as_ushort(inst3_value(inst3_word(x[q], ca.a, ca.b, ca.magic)))
                                                     : __half_as_ushort(onemad_value(onemad_sum(x[q], ca.a, ca.b)));
            } else {
                const int start = 16 * K * r;
                const int w0 = start >> 5;
                const uint32_t W0 = cell[cell_word_index(I, J, w0 % TW, TW)];
                const uint32_t W1 = cell[cell_word_index(I, J, (w0 + 1) % TW, TW)];
                const uint32_t W2 = cell[cell_word_index(I, J, (w0 + 2) % TW, TW)];
                const int off = start & 31;
#pragma unroll
                for (int q = 0; q < 16 / V; ++q) {
                    const uint32_t x = window_general(W0, W1, W2, off + q * K * V);
                    if constexpr (CODE == QTIP_CODE_3INST) {
                        v[q] = __half_as_ushort(inst3_value(inst3_word(x, ca.a, ca.b, ca.magic)));
                    } else if constexpr (CODE == QTIP_CODE_1MAD) {
                        v[q] = __half_as_ushort(onemad_value(onemad_sum(x, ca.a, ca.b)));
                    } else {
                        uint16_t c0, c1;
                        hyb_values(x, lut, ca.Q, ca.two_sign, c0, c1);
                        v[2 * q] = c0;
                        v[2 * q + 1] = c1;
                    }
                }
            }
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                const float w = __half2float(__ushort_as_half(v[c]));
#pragma unroll
                for (int i = 0; i < kSimpleNB; ++i)
                    if (b0 + i < B) acc[i] = fmaf(w, xs[(b0 + i) * kCellCols + J * 16 + c], acc[i]);
            }
        }
#pragma unroll
        for (int i = 0; i < kSimpleNB; ++i)
            if (b0 + i < B) partial[((int64_t)KC * B + b0 + i) * lay.m_pad + row] = acc[i];
    }
}

template <int K, int V, int CODE>
static void launch_simple_t(const Layout& lay, const CodeArgs& ca, const void* packed, const uint16_t* lut,
                            const float* xt, int64_t B, int64_t rb0, int64_t rb1, float* partial, cudaStream_t s) {
    const size_t smem = (size_t)B * kCellCols * sizeof(float);
    auto kern = gemv_simple_kernel<K, V, CODE>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    prefer_max_smem((const void*)kern);
    dim3 grid((unsigned)lay.n_kc, (unsigned)(rb1 - rb0));
    kern<<<grid, 128, smem, s>>>((const uint32_t*)packed, lay, ca, lut, xt, (int)B, rb0, partial);
}

cudaError_t launch_gemv_simple(const Layout& lay, int code, const CodeArgs& ca, const void* packed,
                               const uint16_t* lut, const float* xt, int64_t B, int64_t rb0, int64_t rb1,
                               float* partial, cudaStream_t s) {
#define QTIP_SIMPLE_CASE(KK)                                                                                   \
    case KK:                                                                                                   \
        if (code == QTIP_CODE_3INST) launch_simple_t<KK, 1, QTIP_CODE_3INST>(lay, ca, packed, lut, xt, B, rb0, rb1, partial, s); \
        else if (code == QTIP_CODE_1MAD) launch_simple_t<KK, 1, QTIP_CODE_1MAD>(lay, ca, packed, lut, xt, B, rb0, rb1, partial, s); \
        else launch_simple_t<KK, 2, QTIP_CODE_HYB>(lay, ca, packed, lut, xt, B, rb0, rb1, partial, s);          \
        break;
    switch (lay.k) {
        QTIP_SIMPLE_CASE(1)
        QTIP_SIMPLE_CASE(2)
        QTIP_SIMPLE_CASE(3)
        QTIP_SIMPLE_CASE(4)
        default: return cudaErrorInvalidValue;
    }
#undef QTIP_SIMPLE_CASE
    count_launch(1);
    return cudaGetLastError();
}

}  // namespace qtip
