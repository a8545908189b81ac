// umma_rate.cu -- throughput of tcgen05.mma kind::f16 M=128, K=16 with A from TMEM (the decode-GEMV's
// shape) as a function of N and of the number of independent accumulators.  One CTA per SM, one thread
// issues R MMAs and one commit; cycles from first issue to the mbarrier completion.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../include -o umma_rate umma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2406_11235_b200/csrc/tc.cuh"

using namespace qtip;

template <int N, int NACC, bool A_SMEM>
__global__ void __launch_bounds__(128, 1) rate_kernel(int R, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_holder;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 48 * 1024 / 16; i += 128) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0, 0);
    if (warp == 0) {
        if (threadIdx.x == 0) {
            ptx::mbar_init(ptx::smem_u32(&bar), 1);
            ptx::fence_mbar_init();
        }
        __syncwarp();
        ptx::tmem_alloc(ptx::smem_u32(&tmem_holder), 512);
    }
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_holder;
    constexpr uint32_t idesc = ptx::idesc_f16_f32(128, N);
    if (threadIdx.x == 0) {
        const uint32_t sb = ptx::smem_u32(smem);
        const uint64_t bdesc = ptx::smem_desc_kmajor_noswizzle(sb, 16, 128);
        // A in smem: 128 rows x 16 K, K-major no swizzle: core matrices 8 rows x 16 B; LBO = 128 (K), SBO = 256 (M)
        const uint64_t adesc = ptx::smem_desc_kmajor_noswizzle(sb + 8192, 128, 256);
        const long long t0 = clock64();
        for (int i = 0; i < R; ++i) {
            const uint32_t d = tmem + (uint32_t)((i % NACC) * N);
            if constexpr (A_SMEM) {
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                    "l"(adesc), "l"(bdesc), "r"(idesc), "r"(i >= NACC ? 1u : 0u)
                    : "memory");
            } else {
                ptx::umma_f16_ts(d, tmem + 256u + (uint32_t)(8 * (i % 16)), bdesc, idesc, i >= NACC ? 1u : 0u);
            }
        }
        const long long t1 = clock64();
        ptx::umma_commit(ptx::smem_u32(&bar));
        ptx::mbar_wait(ptx::smem_u32(&bar), 0);
        const long long t2 = clock64();
        if (blockIdx.x == 0) {
            out[0] = (unsigned long long)(t1 - t0);
            out[1] = (unsigned long long)(t2 - t0);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

template <int N, int NACC, bool A_SMEM>
void run(int R, unsigned long long* d) {
    auto k = rate_kernel<N, NACC, A_SMEM>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
    k<<<148, 128, 48 * 1024>>>(R, d);
    k<<<148, 128, 48 * 1024>>>(R, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("N=%3d acc=%d A=%s R=%4d: issue %6llu cyc, complete %6llu cyc -> %.1f cyc/MMA (%s)\n", N, NACC,
           A_SMEM ? "smem" : "tmem", R, h[0], h[1], (double)h[1] / R, cudaGetErrorString(e));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    for (int R : {64, 512}) {
        run<16, 1, false>(R, d);
        run<16, 4, false>(R, d);
        run<16, 1, true>(R, d);
        run<16, 4, true>(R, d);
        run<32, 1, false>(R, d);
        run<64, 1, false>(R, d);
        run<128, 1, false>(R, d);
        run<256, 1, false>(R, d);
        run<64, 1, true>(R, d);
        run<256, 1, true>(R, d);
    }
    return 0;
}
