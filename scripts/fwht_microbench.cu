// fwht_microbench.cu -- cycles of the in-CTA register/shuffle FWHT (fwht.cuh fwht_fast<E>) and of
// the tile readout + fragment writer (park_tiles / tile_read / put_tile), 512 threads, n = 4096,
// measured with clock64 over R back-to-back repetitions inside one CTA (no memory latency).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2406_11235_b200/csrc -o scripts/fwht_microbench scripts/fwht_microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "fwht.cuh"

using namespace qtip::fw;

template <int E>
__global__ void __launch_bounds__(512, 1) bench(float* out, long long* cyc, int a, int R) {
    __shared__ __align__(16) float scr[8192];
    __shared__ __align__(16) uint32_t xs[4096];
    float v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = (float)(threadIdx.x * E + e) * 1e-3f;
    __syncthreads();
    long long t0 = clock64();
    int i0 = 0;
    for (int r = 0; r < R; ++r) i0 += fwht_fast<E>(v, a, scr);
    __syncthreads();
    long long t1 = clock64();
    for (int r = 0; r < R; ++r) {
        park_tiles<E>(v, i0 & 4095, a, scr);
        for (int tile = threadIdx.x; tile < ((1 << a) >> 4); tile += 512) {
            float o[16];
            tile_read<E>(scr, tile, o);
            put_tile<false>(xs + (tile * 16 & 4095), o);
        }
        __syncthreads();
        v[0] += __uint_as_float(xs[threadIdx.x]);
    }
    long long t2 = clock64();
    float acc = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) acc += v[e];
    out[blockIdx.x * 512 + threadIdx.x] = acc + i0;
    if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / R; cyc[1] = (t2 - t1) / R; }
}

int main() {
    float* out; long long* cyc;
    cudaMalloc(&out, 512 * 4 * 148);
    cudaMallocManaged(&cyc, 16);
    for (int rep = 0; rep < 2; ++rep) {
        bench<8><<<1, 512>>>(out, cyc, 12, 64);
        cudaDeviceSynchronize();
    }
    printf("n=4096 E=8 512 thr: fwht_fast %lld cycles, park+tile_read+put_tile %lld cycles\n", cyc[0], cyc[1]);
    bench<8><<<1, 256>>>(out, cyc, 11, 64);
    cudaDeviceSynchronize();
    printf("n=2048 E=8 256 thr: fwht_fast %lld cycles, park+tile_read+put_tile %lld cycles\n", cyc[0], cyc[1]);
    bench<8><<<148, 512>>>(out, cyc, 12, 64);
    cudaDeviceSynchronize();
    printf("n=4096 E=8 148 CTAs: fwht_fast %lld cycles, park+tile_read+put_tile %lld cycles (CTA 0)\n", cyc[0], cyc[1]);
    return 0;
}
