// k_variant.cu -- the code variants of SURVEY §8(f) NEXT-3 on the GPU: decode and fused decode-GEMV
// for
//   * the lookup-only code (QTIP_CODE_LUT): the value of an L-bit state x is
//     LUT[x], a 2^L-entry binary16 table (L = 14: 32 KB -- "too large for current GPU L1 caches, but
//     could fit on near-future hardware"; B200's 228 KB of shared memory per SM holds it), V = 1,
//     T_x x T_y = 32 x 8 (or 16 x 16) blocks, position p = T_y r + c (P:833 row-major scan);
//   * HYB with a 1-D codebook (V = 1, e.g. Q = 6): Alg. 3's hash x^2 + x, index
//     (h >> (15 - Q)) & (2^Q - 1), value LUT[idx] with its sign bit XORed with bit 15 of h.
//
// Device layout (qtip_pack): the usual 128 x 128 cells of 64 sequences; tile (I_l, J_l) of a cell
// (I_l < 128 / T_x, J_l < 128 / T_y) is stored in slot s = I_l (128 / T_y) + J_l, i.e. at the 16 x 16
// position (s / 8, s % 8) of common.cuh's word interleave (for 16 x 16 tiles: the usual layout).
//
// Decode: one CTA per cell, thread = row of the cell, bit-identical to the oracle.  GEMV (the matvec
// path of these codes): one CTA per (row block, 128-column chunk), the whole table staged in shared
// memory, thread = row: decode T_y weights per tile and FFMA against x~ (float32) -- the CUDA-core
// reference structure of impl 1; partial sums per chunk, then the fixed-order reduction.
#include "decode.cuh"
#include "internal.h"

namespace qtip {
namespace {

constexpr int kVNB = 8;                  // batch columns per pass

// T_y weights of row r of tile slot s of a cell: binary16 patterns.
template <int K, int TY, int CODE>
__device__ __forceinline__ void variant_tile_row(const uint32_t* __restrict__ cell, int s, int r, int L, int Q,
                                                 const uint16_t* __restrict__ lut, uint16_t* v) {
    constexpr int TW = 8 * K;
    const int I = s >> 3, J = s & 7;
    const int start = TY * K * r;                      // first stream bit of the row (V = 1)
    const int w0 = start >> 5;
    const uint32_t W0 = cell[cell_word_index(I, J, w0 % TW, TW)];
    const uint32_t W1 = cell[cell_word_index(I, J, (w0 + 1) % TW, TW)];
    const uint32_t W2 = cell[cell_word_index(I, J, (w0 + 2) % TW, TW)];
    const int off = start & 31;
#pragma unroll
    for (int c = 0; c < TY; ++c) {
        const uint32_t w16 = window_general(W0, W1, W2, off + c * K);   // bits [p k, p k + 16) mod kT
        if constexpr (CODE == QTIP_CODE_LUT) {
            v[c] = lut[w16 >> (16 - L)];                                  // the L-bit state
        } else {
            const uint32_t h = w16 * w16 + w16;
            v[c] = (uint16_t)(lut[(h >> (15 - Q)) & ((1u << Q) - 1u)] ^ (h & 0x8000u));
        }
    }
}

template <int K, int TY, int CODE>
__global__ void __launch_bounds__(128) variant_decode_kernel(const uint32_t* __restrict__ packed, Layout lay, int L, int Q,
                                                             const uint16_t* __restrict__ lut, int out_f32, void* out) {
    constexpr int TX = 256 / TY;
    const int KC = blockIdx.x, RB = blockIdx.y, t = threadIdx.x;
    const uint32_t* cell = packed + ((int64_t)RB * lay.n_kc + KC) * lay.cell_words;
    const int64_t row = (int64_t)RB * kCellRows + t;
    if (row >= lay.m) return;
    const int Il = t / TX, r = t % TX;
#pragma unroll 1
    for (int Jl = 0; Jl < kCellCols / TY; ++Jl) {
        const int64_t col0 = (int64_t)KC * kCellCols + Jl * TY;
        if (col0 >= lay.n) break;
        uint16_t v[TY];
        variant_tile_row<K, TY, CODE>(cell, Il * (kCellCols / TY) + Jl, r, L, Q, lut, v);
#pragma unroll
        for (int c = 0; c < TY; ++c) {
            if (out_f32) ((float*)out)[row * lay.n + col0 + c] = __half2float(__ushort_as_half(v[c]));
            else ((uint16_t*)out)[row * lay.n + col0 + c] = v[c];
        }
    }
}

// partial[KC][b][row] = sum over the chunk's columns of W~[row][col] x~[b][col]
template <int K, int TY, int CODE>
__global__ void __launch_bounds__(128) variant_gemv_kernel(const uint32_t* __restrict__ packed, Layout lay, int L, int Q,
                                                           const uint16_t* __restrict__ lut, int lut_n,
                                                           const float* __restrict__ xt, int B, int64_t rb0,
                                                           float* __restrict__ partial) {
    constexpr int TX = 256 / TY;
    extern __shared__ __align__(16) uint8_t vsm[];
    uint16_t* slut = reinterpret_cast<uint16_t*>(vsm);                      // the whole table
    float* xs = reinterpret_cast<float*>(vsm + ((2 * lut_n + 15) & ~15));   // [B][128] slice of x~
    const int KC = blockIdx.x;
    const int64_t RB = rb0 + blockIdx.y;
    const int t = threadIdx.x;
    for (int e = t; e < lut_n / 8; e += 128) reinterpret_cast<uint4*>(slut)[e] = __ldg(reinterpret_cast<const uint4*>(lut) + e);
    for (int e = t; e < B * kCellCols; e += 128) {
        const int b = e / kCellCols, c = e % kCellCols;
        const int64_t col = (int64_t)KC * kCellCols + c;
        xs[e] = col < lay.n ? xt[(int64_t)b * lay.n_pad + col] : 0.0f;
    }
    __syncthreads();
    const uint32_t* cell = packed + (RB * lay.n_kc + KC) * lay.cell_words;
    const int64_t row = RB * kCellRows + t;
    const int Il = t / TX, r = t % TX;
    for (int b0 = 0; b0 < B; b0 += kVNB) {
        float acc[kVNB];
#pragma unroll
        for (int i = 0; i < kVNB; ++i) acc[i] = 0.0f;
#pragma unroll 1
        for (int Jl = 0; Jl < kCellCols / TY; ++Jl) {
            uint16_t v[TY];
            variant_tile_row<K, TY, CODE>(cell, Il * (kCellCols / TY) + Jl, r, L, Q, slut, v);
#pragma unroll
            for (int c = 0; c < TY; ++c) {
                const float w = __half2float(__ushort_as_half(v[c]));
#pragma unroll
                for (int i = 0; i < kVNB; ++i)
                    if (b0 + i < B) acc[i] = fmaf(w, xs[(b0 + i) * kCellCols + Jl * TY + c], acc[i]);
            }
        }
#pragma unroll
        for (int i = 0; i < kVNB; ++i)
            if (b0 + i < B) partial[((int64_t)KC * B + b0 + i) * lay.m_pad + row] = acc[i];
    }
}

int variant_lut_entries(const qtip_params* p) { return p->code == QTIP_CODE_LUT ? 1 << p->L : 1 << p->Q; }

}  // namespace

bool is_variant(const qtip_params* p) { return p->code == QTIP_CODE_LUT || (p->code == QTIP_CODE_HYB && p->V == 1); }

#define QTIP_VARIANT_DISPATCH(LAUNCH)                                                                           \
    do {                                                                                                        \
        const bool lutc = p->code == QTIP_CODE_LUT;                                                             \
        const int ty = p->Ty;                                                                                   \
        switch (lay.k * 100 + ty * 10 + (lutc ? 1 : 0)) {                                                       \
            case 1 * 100 + 160 + 1: LAUNCH(1, 16, QTIP_CODE_LUT); break;                                        \
            case 2 * 100 + 160 + 1: LAUNCH(2, 16, QTIP_CODE_LUT); break;                                        \
            case 3 * 100 + 160 + 1: LAUNCH(3, 16, QTIP_CODE_LUT); break;                                        \
            case 4 * 100 + 160 + 1: LAUNCH(4, 16, QTIP_CODE_LUT); break;                                        \
            case 1 * 100 + 80 + 1: LAUNCH(1, 8, QTIP_CODE_LUT); break;                                          \
            case 2 * 100 + 80 + 1: LAUNCH(2, 8, QTIP_CODE_LUT); break;                                          \
            case 3 * 100 + 80 + 1: LAUNCH(3, 8, QTIP_CODE_LUT); break;                                          \
            case 4 * 100 + 80 + 1: LAUNCH(4, 8, QTIP_CODE_LUT); break;                                          \
            case 1 * 100 + 160: LAUNCH(1, 16, QTIP_CODE_HYB); break;                                            \
            case 2 * 100 + 160: LAUNCH(2, 16, QTIP_CODE_HYB); break;                                            \
            case 3 * 100 + 160: LAUNCH(3, 16, QTIP_CODE_HYB); break;                                            \
            case 4 * 100 + 160: LAUNCH(4, 16, QTIP_CODE_HYB); break;                                            \
            default: return cudaErrorInvalidValue;                                                              \
        }                                                                                                       \
    } while (0)

cudaError_t launch_variant_decode(const qtip_params* p, const Layout& lay, const void* packed, const uint16_t* lut,
                                  int out_f32, void* out, cudaStream_t s) {
    dim3 grid((unsigned)lay.n_kc, (unsigned)lay.n_rb);
#define QTIP_VDEC(KK, TYY, CC) \
    variant_decode_kernel<KK, TYY, CC><<<grid, 128, 0, s>>>((const uint32_t*)packed, lay, p->L, p->Q, lut, out_f32, out)
    QTIP_VARIANT_DISPATCH(QTIP_VDEC);
#undef QTIP_VDEC
    count_launch(1);
    return cudaGetLastError();
}

cudaError_t launch_variant_gemv(const qtip_params* p, const Layout& lay, const void* packed, const uint16_t* lut,
                                const float* xt, int64_t B, int64_t rb0, int64_t rb1, float* partial, cudaStream_t s) {
    const int lut_n = variant_lut_entries(p);
    const size_t smem = (size_t)((2 * lut_n + 15) & ~15) + (size_t)B * kCellCols * 4;
    dim3 grid((unsigned)lay.n_kc, (unsigned)(rb1 - rb0));
    cudaError_t e = cudaSuccess;
#define QTIP_VGEMV(KK, TYY, CC)                                                                                  \
    {                                                                                                         \
        auto kern = variant_gemv_kernel<KK, TYY, CC>;                                                         \
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);              \
        if (e == cudaSuccess)                                                                                 \
            kern<<<grid, 128, smem, s>>>((const uint32_t*)packed, lay, p->L, p->Q, lut, lut_n, xt, (int)B, rb0, \
                                         partial);                                                            \
    }
    QTIP_VARIANT_DISPATCH(QTIP_VGEMV);
#undef QTIP_VGEMV
    if (e != cudaSuccess) return e;
    count_launch(1);
    return cudaGetLastError();
}

size_t variant_gemv_smem(const qtip_params* p, int64_t B) {
    return (size_t)((2 * variant_lut_entries(p) + 15) & ~15) + (size_t)B * kCellCols * 4;
}

}  // namespace qtip
