// Debug aid: (1) tcgen05.mma SS (A and B from smem) issue cost vs TS; (2) mma.sync m16n8k16 throughput.
#include <cstdio>
#include <cstdint>
#include "tc.cuh"
using namespace qtip;

__device__ __forceinline__ void umma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

__global__ void bench_ss(int n_mma, int N, long long* out) {
    __shared__ __align__(1024) uint8_t sm[32768];
    __shared__ uint64_t bar;
    __shared__ uint32_t holder;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 32768 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) { ptx::mbar_init(ptx::smem_u32(&bar), 1); ptx::fence_mbar_init(); }
    if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&holder), 512);
    ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
    const uint32_t tmem = holder;
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t adesc = ptx::smem_desc_kmajor_noswizzle(ptx::smem_u32(sm), 128u, 256u);
    const uint64_t bdesc = ptx::smem_desc_kmajor_noswizzle(ptx::smem_u32(sm) + 16384, 128u, 256u);
    if (warp == 0) {
        for (int rep = 0; rep < 3; ++rep) {
            long long t0 = clock64();
            if (ptx::elect_one()) {
#pragma unroll 8
                for (int i = 0; i < n_mma; ++i) umma_ss(tmem, adesc, bdesc, idesc, 1);
                ptx::umma_commit(ptx::smem_u32(&bar));
            }
            __syncwarp();
            ptx::mbar_wait(ptx::smem_u32(&bar), rep & 1);
            long long t2 = clock64();
            if (threadIdx.x == 0 && rep == 2) out[0] = t2 - t0;
        }
    }
    ptx::tc_fence_before(); __syncthreads();
    if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}

__global__ void bench_ts_unrolled(int n_mma, int N, long long* out) {
    __shared__ __align__(1024) uint8_t sm[16384];
    __shared__ uint64_t bar;
    __shared__ uint32_t holder;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 16384 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) { ptx::mbar_init(ptx::smem_u32(&bar), 1); ptx::fence_mbar_init(); }
    if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&holder), 512);
    ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
    const uint32_t tmem = holder;
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t bdesc = ptx::smem_desc_kmajor_noswizzle(ptx::smem_u32(sm), 128u, 256u);
    if (warp == 0) {
        for (int rep = 0; rep < 3; ++rep) {
            long long t0 = clock64();
            if (ptx::elect_one()) {
#pragma unroll 8
                for (int i = 0; i < n_mma; ++i) ptx::umma_f16_ts(tmem, tmem + 256, bdesc, idesc, 1);
                ptx::umma_commit(ptx::smem_u32(&bar));
            }
            __syncwarp();
            ptx::mbar_wait(ptx::smem_u32(&bar), rep & 1);
            long long t2 = clock64();
            if (threadIdx.x == 0 && rep == 2) out[0] = t2 - t0;
        }
    }
    ptx::tc_fence_before(); __syncthreads();
    if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}

__global__ void bench_hmma(int iters, long long* out, float* sink) {
    uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 9, b1 = a0 ^ 5;
    float c[8][4] = {};
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    long long t1 = clock64();
    float s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

int main() {
    long long* d; float* sink;
    cudaMalloc(&d, 16); cudaMalloc(&sink, 1 << 24);
    for (int N : {16, 64, 256}) for (int n : {16, 64, 256}) {
        long long h;
        bench_ss<<<1, 128>>>(n, N, d); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("SS  N=%3d n=%3d total=%6lld per-mma=%.1f cyc  %s\n", N, n, h, (double)h / n, cudaGetErrorString(cudaGetLastError()));
        bench_ts_unrolled<<<1, 128>>>(n, N, d); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("TS  N=%3d n=%3d total=%6lld per-mma=%.1f cyc  %s\n", N, n, h, (double)h / n, cudaGetErrorString(cudaGetLastError()));
    }
    for (int warps : {1, 4, 8, 16}) {
        long long h; int iters = 1000;
        bench_hmma<<<1, 32 * warps>>>(iters, d, sink); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("HMMA.16816.F32 warps/SM=%2d: %.2f cyc per HMMA per warp -> %.2f HMMA/clk/SM  %s\n", warps,
               (double)h / (iters * 8), warps * iters * 8.0 / h, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
