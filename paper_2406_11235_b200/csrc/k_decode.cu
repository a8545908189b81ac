// k_decode.cu -- qtip_decode: packed tiles -> dense W~ (binary16 or float32), bit-exact.
//
// One CTA per 128 x 256 cell, one thread per output row of the cell; each thread decodes
// its row of all 16 tiles of the cell (16 contiguous windows per tile, see decode.cuh).
#include "decode.cuh"
#include "internal.h"

namespace qtip {

template <int K, int V, int CODE>
__device__ __forceinline__ void decode_tile_row(const uint32_t* __restrict__ cell, int I, int J, int r,
                                                const CodeArgs& ca, const uint16_t* __restrict__ lut,
                                                uint16_t out[16]) {
    constexpr int TW = 8 * K;
    if constexpr (K == 2 && V == 1) {
        const uint32_t A = cell[cell_word_index(I, J, r, TW)];
        const uint32_t B = cell[cell_word_index(I, J, (r + 1) & 15, TW)];
        uint32_t x[16];
        windows_k2v1(A, B, x);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            if constexpr (CODE == QTIP_CODE_3INST) {
                out[q] = __half_as_ushort(inst3_value(inst3_word(x[q], ca.a, ca.b, ca.magic)));
            } else {
                out[q] = __half_as_ushort(onemad_value(onemad_sum(x[q], ca.a, ca.b)));
            }
        }
    } else {
        const int start = 16 * K * r;                    // first bit of the row
        const int w0 = start >> 5;
        const uint32_t W0 = cell[cell_word_index(I, J, w0 % TW, TW)];
        const uint32_t W1 = cell[cell_word_index(I, J, (w0 + 1) % TW, TW)];
        const uint32_t W2 = cell[cell_word_index(I, J, (w0 + 2) % TW, TW)];
        const int off = start & 31;
#pragma unroll
        for (int q = 0; q < 16 / V; ++q) {
            const uint32_t x = window_general(W0, W1, W2, off + q * K * V);
            if constexpr (CODE == QTIP_CODE_3INST) {
                out[q] = __half_as_ushort(inst3_value(inst3_word(x, ca.a, ca.b, ca.magic)));
            } else if constexpr (CODE == QTIP_CODE_1MAD) {
                out[q] = __half_as_ushort(onemad_value(onemad_sum(x, ca.a, ca.b)));
            } else {
                uint16_t c0, c1;
                hyb_values(x, lut, ca.Q, ca.two_sign, c0, c1);
                out[2 * q] = c0;
                out[2 * q + 1] = c1;
            }
        }
    }
}

template <int K, int V, int CODE>
__global__ void __launch_bounds__(128) decode_kernel(const uint32_t* __restrict__ packed, Layout lay, CodeArgs ca,
                                                     const uint16_t* __restrict__ lut, int out_f32, void* out) {
    const int KC = blockIdx.x, RB = blockIdx.y;
    const int t = threadIdx.x, I = t >> 4, r = t & 15;
    const uint32_t* cell = packed + ((int64_t)RB * lay.n_kc + KC) * lay.cell_words;
    const int64_t row = (int64_t)RB * kCellRows + t;
    if (row >= lay.m) return;
#pragma unroll 1
    for (int J = 0; J < kCellTileCols; ++J) {
        const int64_t col0 = (int64_t)KC * kCellCols + J * kTile;
        if (col0 >= lay.n) break;
        uint16_t v[16];
        decode_tile_row<K, V, CODE>(cell, I, J, r, ca, lut, v);
        if (out_f32) {
            float4* o = reinterpret_cast<float4*>((float*)out + row * lay.n + col0);
#pragma unroll
            for (int c = 0; c < 4; ++c)
                o[c] = make_float4(__half2float(__ushort_as_half(v[4 * c])), __half2float(__ushort_as_half(v[4 * c + 1])),
                                   __half2float(__ushort_as_half(v[4 * c + 2])), __half2float(__ushort_as_half(v[4 * c + 3])));
        } else {
            uint4* o = reinterpret_cast<uint4*>((uint16_t*)out + row * lay.n + col0);
#pragma unroll
            for (int c = 0; c < 2; ++c)
                o[c] = make_uint4(v[8 * c] | ((uint32_t)v[8 * c + 1] << 16), v[8 * c + 2] | ((uint32_t)v[8 * c + 3] << 16),
                                  v[8 * c + 4] | ((uint32_t)v[8 * c + 5] << 16), v[8 * c + 6] | ((uint32_t)v[8 * c + 7] << 16));
        }
    }
}

template <int K, int V, int CODE>
static void launch_decode_t(const Layout& lay, const CodeArgs& ca, const void* packed, const uint16_t* lut, int out_f32,
                            void* out, cudaStream_t s) {
    dim3 grid((unsigned)lay.n_kc, (unsigned)lay.n_rb);
    decode_kernel<K, V, CODE><<<grid, 128, 0, s>>>((const uint32_t*)packed, lay, ca, lut, out_f32, out);
}

cudaError_t launch_decode(const Layout& lay, int code, int V, const CodeArgs& ca, const void* packed,
                          const uint16_t* lut, int out_f32, void* out, cudaStream_t s) {
#define QTIP_DEC_CASE(KK)                                                                    \
    case KK:                                                                                 \
        if (code == QTIP_CODE_3INST) launch_decode_t<KK, 1, QTIP_CODE_3INST>(lay, ca, packed, lut, out_f32, out, s); \
        else if (code == QTIP_CODE_1MAD) launch_decode_t<KK, 1, QTIP_CODE_1MAD>(lay, ca, packed, lut, out_f32, out, s); \
        else launch_decode_t<KK, 2, QTIP_CODE_HYB>(lay, ca, packed, lut, out_f32, out, s);                \
        break;
    switch (lay.k) {
        QTIP_DEC_CASE(1)
        QTIP_DEC_CASE(2)
        QTIP_DEC_CASE(3)
        QTIP_DEC_CASE(4)
        default: return cudaErrorInvalidValue;
    }
#undef QTIP_DEC_CASE
    (void)V;
    count_launch(1);
    return cudaGetLastError();
}

}  // namespace qtip
