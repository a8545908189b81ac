// decode_microbench.cu -- steady-state rate of the register-fed decode-MMA inner loop (mma_tile.cuh
// tile_pair, 3INST k = 2, batch 1) on one SM with the weights already in shared memory: weights per
// clock per SM for 8 / 16 / 32 warps.  Separates the decode loop's own throughput from the
// layer kernel's prologue, x~ and epilogue phases.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../include -o decode_microbench decode_microbench.cu
#include <cstdio>

#include "../paper_2406_11235_b200/csrc/mma_tile.cuh"
#include "../paper_2406_11235_b200/csrc/tc.cuh"

using namespace qtip;
using namespace qtip::mma;

constexpr int N_IT = 256;

// MODE 0: tile_pair (decode + HMMA); 1: HMMA only (A = raw stream words); 2: decode only (the
// 3INST words are folded into fp32 adds instead of HMMAs); 3: decode + tcgen05.st of the A words
// into TMEM (the tcgen05 path's data movement, no MMA)
template <int NACC, int MODE = 0>
__global__ void loop(const uint32_t* __restrict__ src, float* out, long long* cyc) {
    __shared__ __align__(16) uint32_t chunk[8 * 4 * 64];  // 8 units x 4 tile pairs (k = 2: 32 words each)
    __shared__ __align__(16) uint32_t xs[8 * 128];         // x~ of 8 x 8 tiles (fragment order, K-doubled)
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) chunk[i] = src[i & 1023];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) xs[i] = 0x3c003c00u;
    __syncthreads();
    const int lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
    CodeArgs ca;
    ca.a = 89226354u;
    ca.b = 64248484u;
    ca.magic = 0x3B603B60u;
    ca.Q = 9;
    ca.two_sign = 0;
    const Lcg<QTIP_CODE_3INST, true> lcg(ca);
    float acc[NACC][1][4] = {};
    __shared__ uint32_t tmem_base;
    if (MODE == 3) {
        if (threadIdx.x < 32) ptx::tmem_alloc(ptx::smem_u32(&tmem_base), 64);
        ptx::tc_fence_before();
        __syncthreads();
        ptx::tc_fence_after();
    }
    const uint32_t tcol = MODE == 3 ? tmem_base + (((threadIdx.x >> 5) & 3) << 21) : 0u;
    const long long t0 = clock64();
    for (int it = 0; it < N_IT; ++it) {
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) {
            uint32_t bf[2][1][4];
            const int ub = (it + (threadIdx.x >> 5)) & 7;            // a different unit every iteration (no hoisting)
            load_bfrag<1, false>(xs + 128 * ub, 128, 2 * pp, g, tig, 1, bf[0]);
            load_bfrag<1, false>(xs + 128 * ub, 128, 2 * pp + 1, g, tig, 1, bf[1]);
            if constexpr (MODE == 0) {
                tile_pair<2, QTIP_CODE_3INST, 1, true>(chunk + 256 * ub + pp * 32, bf, acc[pp % NACC], g, tig, lcg, ca, nullptr);
            } else if constexpr (MODE == 1) {
                const uint4 w = *reinterpret_cast<const uint4*>(chunk + pp * 32 + 4 * g);
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    hmma_16816(acc[pp % NACC][0], w.x, w.y, w.z, w.w, bf[t][0][0], bf[t][0][1]);
                    hmma_16816(acc[pp % NACC][0], w.y, w.z, w.w, w.x, bf[t][0][2], bf[t][0][3]);
                }
            } else {
                uint4 w01;
                uint2 w2;
                const uint32_t a0 = ptx::smem_u32(chunk + pp * 32 + 4 * g + (it & 1) * 128);
                const uint32_t a1 = ptx::smem_u32(chunk + pp * 32 + 2 * ((2 * g + 2) & 15) + (it & 1) * 128);
                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w01.x), "=r"(w01.y), "=r"(w01.z), "=r"(w01.w) : "r"(a0));
                asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(w2.x), "=r"(w2.y) : "r"(a1));
                uint32_t zz[8];
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const uint32_t W0 = t ? w01.y : w01.x, W1 = t ? w01.w : w01.z, W2 = t ? w2.y : w2.x;
                    const uint32_t F[4] = {__funnelshift_l(W1, W0, 4 * tig), __funnelshift_l(W1, W0, 4 * tig + 2),
                                           __funnelshift_l(W2, W1, 4 * tig), __funnelshift_l(W2, W1, 4 * tig + 2)};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint32_t zh, zl;
                        lcg_pair<QTIP_CODE_3INST, true, true>(F[q], lcg, ca.magic, zh, zl);
                        if constexpr (MODE == 2) acc[pp % NACC][0][q] += __uint_as_float(zh) + __uint_as_float(zl);
                        zz[2 * q] = zh;
                        zz[2 * q + 1] = zl;
                    }
                    if constexpr (MODE == 3) ptx::tmem_st8(tcol + 8 * t, zz);
                }
            }
        }
    }
    if (MODE == 3) ptx::tc_wait_st();
    const long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < NACC; ++q) s += acc[q][0][0] + acc[q][0][1] + acc[q][0][2] + acc[q][0][3];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) *cyc = t1 - t0;
    if (MODE == 3) {
        ptx::tc_fence_before();
        __syncthreads();
        if (threadIdx.x < 32) ptx::tmem_dealloc(tmem_base, 64);
    }
}

int main() {
    uint32_t* src;
    float* out;
    long long* c;
    cudaMalloc(&src, 4096);
    cudaMalloc(&out, 4096 * 4);
    cudaMalloc(&c, 8);
    uint32_t h[1024];
    for (int i = 0; i < 1024; ++i) h[i] = 0x9E3779B9u * (i + 1);
    cudaMemcpy(src, h, 4096, cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 4; ++mode)
    for (int warps : {16, 32}) {
        for (int nacc : {2}) {
            auto k = mode == 0 ? loop<2, 0> : (mode == 1 ? loop<2, 1> : (mode == 2 ? loop<2, 2> : loop<2, 3>));
            k<<<1, 32 * warps>>>(src, out, c);
            k<<<1, 32 * warps>>>(src, out, c);
            long long cy;
            cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
            const double weights = (double)warps * N_IT * 4 * 512;   // 4 pairs x 2 tiles x 256 per warp-iteration
            printf("mode=%d warps=%2d acc=%d: %.1f weights/clk/SM (%lld cycles)\n", mode, warps, nacc, weights / cy, cy);
        }
    }
    return 0;
}
