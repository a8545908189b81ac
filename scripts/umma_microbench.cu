// Microbenchmark (debug aid, not part of libqtip): latency / throughput of tcgen05.mma
// kind::f16 M=128, A from TMEM, B from shared memory, for N in {16, 64, 256}; chains into one
// D accumulator vs. round-robin over 4 accumulators; and the commit -> mbarrier round trip.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2406_11235_b200/csrc umma_microbench.cu
#include <cstdio>
#include <cstdint>
#include "tc.cuh"

using namespace qtip;

__global__ void bench(int n_mma, int N, int ndist, long long* out) {
    __shared__ __align__(1024) uint8_t bsm[16384];
    __shared__ uint64_t bar;
    __shared__ uint32_t holder;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 16384 / 16; i += blockDim.x) reinterpret_cast<uint4*>(bsm)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) { ptx::mbar_init(ptx::smem_u32(&bar), 1); ptx::fence_mbar_init(); }
    if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&holder), 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = holder;
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    if (warp == 0) {
        for (int rep = 0; rep < 3; ++rep) {
            long long t0 = clock64();
            if (ptx::elect_one()) {
                for (int i = 0; i < n_mma; ++i) {
                    const uint32_t start = ptx::smem_u32(bsm) + (i % 8) * 512;
                    const uint64_t bdesc = ptx::smem_desc_kmajor_noswizzle(start, 128u, 256u);
                    const uint32_t d = tmem + (uint32_t)((i % ndist) * N);
                    ptx::umma_f16_ts(d, tmem + 256 + (i % 8) * 8, bdesc, idesc, i >= ndist);
                }
                ptx::umma_commit(ptx::smem_u32(&bar));
            }
            __syncwarp();
            long long t1 = clock64();
            ptx::mbar_wait(ptx::smem_u32(&bar), rep & 1);
            long long t2 = clock64();
            if (threadIdx.x == 0 && rep == 2) { out[0] = t1 - t0; out[1] = t2 - t0; }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}

int main() {
    long long* d;
    cudaMalloc(&d, 16);
    for (int N : {16, 64, 128}) {
        for (int ndist : {1, 4}) {
            for (int n : {1, 4, 16, 64, 256}) {
                bench<<<1, 128>>>(n, N, ndist, d);
                long long h[2];
                cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
                cudaError_t e = cudaGetLastError();
                printf("N=%3d accum=%d n_mma=%3d issue=%6lld cyc  issue+complete=%6lld cyc  per-mma=%.1f  %s\n", N, ndist,
                       n, h[0], h[1], (double)h[1] / n, cudaGetErrorString(e));
            }
        }
    }
    return 0;
}
