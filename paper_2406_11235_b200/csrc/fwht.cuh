// fwht.cuh -- in-CTA Walsh-Hadamard transform of a power-of-two vector held in registers (shared by
// the fused layer kernel k_layer.cu and the single-CTA RHT kernel of k_rht.cu), plus the tile-wise
// readout and the binary16 B-fragment writer of x~.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

namespace qtip {
namespace fw {

// Register/shuffle Walsh-Hadamard transform of one length-n = 2^a vector held by T = n / E threads
// (layout A: thread t owns elements t E + e).  Butterflies on the E register bits and the 5 lane
// bits run without memory traffic; if warps hold further bits, one swizzled shared-memory
// transpose (scr: n floats) swaps the warp field into the lanes and those bits run as shuffles.
// Every thread of the CTA must call it (it synchronises); threads >= T carry don't-care values.
// Returns the index of the thread's first element afterwards (E contiguous elements).
template <int E>
__device__ __forceinline__ int fwht_fast(float (&v)[E], int a, float* scr) {
    constexpr int s = E == 4 ? 2 : (E == 8 ? 3 : 4);
    const int t = threadIdx.x, lane = t & 31;
    const int T = (1 << a) >> s;
#pragma unroll
    for (int h = 1; h < E; h <<= 1)
#pragma unroll
        for (int e = 0; e < E; ++e)
            if (!(e & h)) {
                const float x0 = v[e], x1 = v[e | h];
                v[e] = x0 + x1;
                v[e | h] = x0 - x1;
            }
    // shuffle butterflies: (lane & h) ? o - v : v + o  ==  fma(v, +-1, o), one rounding either way
    const int lb = a - s < 5 ? a - s : 5;
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        if (j < lb) {
            const int h = 1 << j;
            const float sg = (lane & h) ? -1.0f : 1.0f;
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = fmaf(v[e], sg, __shfl_xor_sync(0xffffffffu, v[e], h));
        }
    }
    const int wb = a - s - 5;
    if (wb <= 0) return t * E;
    // transpose: float4 slot q = i >> 2 stored at q ^ (warp field & 7)
    auto slot = [&](int i) { return ((i >> 2) ^ ((i >> (s + 5)) & 7)) << 2; };
    if (t < T) {
#pragma unroll
        for (int e = 0; e < E; e += 4)
            *reinterpret_cast<float4*>(scr + slot(t * E + e)) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
    }
    __syncthreads();
    const int w2 = t >> 5;                                          // = the old lane's high wb bits
    const int wo = lane >> (5 - wb), llo = lane & ((1 << (5 - wb)) - 1);
    const int i0 = (wo << (s + 5)) | (w2 << (s + 5 - wb)) | (llo << s);
    if (t < T) {
#pragma unroll
        for (int e = 0; e < E; e += 4) {
            const float4 q = *reinterpret_cast<const float4*>(scr + slot(i0 + e));
            v[e] = q.x; v[e + 1] = q.y; v[e + 2] = q.z; v[e + 3] = q.w;
        }
    }
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        if (j < wb) {
            const int h = 1 << (5 - wb + j);
            const float sg = (lane & h) ? -1.0f : 1.0f;
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = fmaf(v[e], sg, __shfl_xor_sync(0xffffffffu, v[e], h));
        }
    }
    __syncthreads();                                                // scr may be reused
    return i0;
}

// After fwht_fast: park the thread's E values (first index i0) in scr with the transpose swizzle,
// so that whole 16-element tiles can be read back conflict-free by one thread each (tile_read).
template <int E>
__device__ __forceinline__ void park_tiles(const float (&v)[E], int i0, int a, float* scr) {
    constexpr int s = E == 4 ? 2 : (E == 8 ? 3 : 4);
    const int T = (1 << a) >> s;
    if ((int)threadIdx.x < T) {
#pragma unroll
        for (int e = 0; e < E; e += 4) {
            const int i = i0 + e;
            *reinterpret_cast<float4*>(scr + (((i >> 2) ^ ((i >> (s + 5)) & 7)) << 2)) =
                make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
        }
    }
    __syncthreads();
}
// the 16 values of tile `tile` (elements 16 tile .. 16 tile + 15) parked by park_tiles<E>; with
// consecutive tiles on consecutive lanes the swizzle spreads each 16-B read over the bank groups
template <int E>
__device__ __forceinline__ void tile_read(const float* scr, int tile, float (&o)[16]) {
    constexpr int s = E == 4 ? 2 : (E == 8 ? 3 : 4);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int i = 16 * tile + 4 * j;
        const float4 q = *reinterpret_cast<const float4*>(scr + (((i >> 2) ^ ((i >> (s + 5)) & 7)) << 2));
        o[4 * j] = q.x; o[4 * j + 1] = q.y; o[4 * j + 2] = q.z; o[4 * j + 3] = q.w;
    }
}
// one tile of x~ (16 values, already scaled) -> binary16 B-fragment words at dst (16 words
// K-doubled, 8 words HYB); the 16-B chunks go out in a lane-rotated order (consecutive lanes write
// consecutive tiles, 64 B apart: rotation spreads a store instruction over 8 bank groups)
template <bool kHyb, bool kSwap = false>
__device__ __forceinline__ void put_tile(uint32_t* dst, const float (&v)[16]) {
    // one packed f32x2 -> f16x2 conversion (round to nearest) per word; low half = first argument
    auto h2 = [&](float lo, float hi) {
        const __half2 q = __floats2half2_rn(lo, hi);
        return *reinterpret_cast<const uint32_t*>(&q);
    };
    if constexpr (!kHyb) {
        uint4 w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {                               // words 4j..4j+3 = cols 2j, 2j+8, 2j+1, 2j+9
            w[j] = make_uint4(h2(v[2 * j], v[2 * j]), h2(v[2 * j + 8], v[2 * j + 8]), h2(v[2 * j + 1], v[2 * j + 1]),
                              h2(v[2 * j + 9], v[2 * j + 9]));
        }
        const int r = (threadIdx.x >> 1) & 3;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const int j = (jj + r) & 3;
            const uint4 x = j == 0 ? w[0] : (j == 1 ? w[1] : (j == 2 ? w[2] : w[3]));
            *reinterpret_cast<uint4*>(dst + 4 * j) = x;
        }
    } else {
        uint4 w[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {                               // word ww holds pair 4 (ww & 1) + (ww >> 1)
            uint32_t u[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int ww = 4 * j + k, pr = 4 * (ww & 1) + (ww >> 1);
                u[k] = kSwap ? h2(v[2 * pr + 1], v[2 * pr]) : h2(v[2 * pr], v[2 * pr + 1]);
            }
            w[j] = make_uint4(u[0], u[1], u[2], u[3]);
        }
        const int r = (threadIdx.x >> 2) & 1;
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const int j = jj ^ r;
            *reinterpret_cast<uint4*>(dst + 4 * j) = j ? w[1] : w[0];
        }
    }
}

// fast-path element count per thread for a power-of-two length n (0: not supported)
__host__ __device__ inline int fwht_fast_E(int64_t n, int a, int threads) {
    if (n != ((int64_t)1 << a) || n < 128) return 0;
    const int64_t E = n / threads < 4 ? 4 : n / threads;
    return (E == 4 || E == 8 || E == 16) ? (int)E : 0;
}


}  // namespace fw
}  // namespace qtip
