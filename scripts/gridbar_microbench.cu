// gridbar_microbench.cu -- cost of an in-kernel grid barrier (all CTAs co-resident, one per SM)
// versus a kernel boundary (back-to-back launches in a CUDA graph, with and without PDL).
// Decides whether the fused layer kernel (k_layer.cu) should replace kernel boundaries by
// in-kernel barriers.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridbar gridbar_microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint64_t gtime() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__device__ __forceinline__ void grid_barrier(unsigned int* ctr, unsigned int P) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int old;
        asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
        const unsigned int target = (old / P + 1) * P;
        const uint64_t t0 = gtime();
        while (true) {
            unsigned int v;
            asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
            if ((int)(v - target) >= 0) break;
            if (gtime() - t0 > 2000000000ull) __trap();
        }
    }
    __syncthreads();
}

// flag-array barrier (k_layer.cu grid_sync): per-CTA epoch words, one warp polls them all
__device__ __forceinline__ void flag_barrier(unsigned* flags, unsigned e) {
    __syncthreads();
    if (threadIdx.x < 32) {
        if (threadIdx.x == 0) {
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x), "r"(e) : "memory");
        }
        const uint64_t t0 = gtime();
        for (int j = threadIdx.x; j < (int)gridDim.x; j += 32) {
            while (true) {
                unsigned v;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + j) : "memory");
                if ((int)(v - e) >= 0) break;
                if (gtime() - t0 > 2000000000ull) __trap();
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// split-line counter barrier (k_layer.cu grid_sync): arrival counter and generation word on
// different 128-B lines, relaxed polling of the generation, one fence after
template <int SLEEP>
__device__ __forceinline__ void split_barrier(unsigned* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned* cnt = bar;
        unsigned* gen = bar + 32;
        unsigned g, old;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(gen) : "memory");
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
        if (old == gridDim.x - 1) {
            asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(cnt) : "memory");
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(g + 1) : "memory");
        } else {
            const uint64_t t0 = gtime();
            while (true) {
                unsigned v;
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gen) : "memory");
                if (v != g) break;
                if (SLEEP) __nanosleep(SLEEP);
                if (gtime() - t0 > 2000000000ull) __trap();
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
    }
    __syncthreads();
}

template <int SLEEP>
__global__ void __launch_bounds__(512, 1) split_kernel(unsigned* bar, int R, float* sink) {
    float acc = 0.f;
    for (int r = 0; r < R; ++r) {
        acc += threadIdx.x * 1e-9f;
        split_barrier<SLEEP>(bar);
    }
    if (acc == 12345.f) sink[0] = acc;
}

__global__ void __launch_bounds__(512, 1) flag_kernel(unsigned* flags, int R, float* sink) {
    unsigned e = __ldcg(flags + blockIdx.x);
    float acc = 0.f;
    for (int r = 0; r < R; ++r) {
        acc += threadIdx.x * 1e-9f;
        flag_barrier(flags, ++e);
    }
    if (acc == 12345.f) sink[0] = acc;
}

__global__ void __launch_bounds__(512, 1) bar_kernel(unsigned int* ctr, int R, float* sink) {
    const unsigned int P = gridDim.x;
    float acc = 0.f;
    for (int r = 0; r < R; ++r) {
        acc += threadIdx.x * 1e-9f;
        grid_barrier(ctr, P);
    }
    if (acc == 12345.f) sink[0] = acc;
}

__global__ void __launch_bounds__(512, 1) empty_kernel(float* sink, int pdl) {
    if (pdl) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
    if (threadIdx.x == 9999) sink[blockIdx.x] = 1.f;
}

int main() {
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    unsigned int* ctr;
    float* sink;
    CK(cudaMalloc(&ctr, 4));
    CK(cudaMemset(ctr, 0, 4));
    CK(cudaMalloc(&sink, 4096 * 4));
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int P : {sms, 2 * sms}) {
        if (P == 2 * sms) {
            // 2 CTAs of 256 threads per SM
        }
        const int R = 2000;
        const int thr = P == sms ? 512 : 256;
        bar_kernel<<<P, thr, 0, s>>>(ctr, 10, sink);
        CK(cudaStreamSynchronize(s));
        CK(cudaEventRecord(e0, s));
        bar_kernel<<<P, thr, 0, s>>>(ctr, R, sink);
        CK(cudaEventRecord(e1, s));
        CK(cudaStreamSynchronize(s));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("grid barrier: P=%d CTAs x %d thr: %.3f us per barrier\n", P, thr, 1e3f * ms / R);
    }
    {
        unsigned* flags;
        CK(cudaMalloc(&flags, 4096));
        CK(cudaMemset(flags, 0, 4096));
        const int R = 2000;
        flag_kernel<<<sms, 512, 0, s>>>(flags, 10, sink);
        CK(cudaStreamSynchronize(s));
        CK(cudaEventRecord(e0, s));
        flag_kernel<<<sms, 512, 0, s>>>(flags, R, sink);
        CK(cudaEventRecord(e1, s));
        CK(cudaStreamSynchronize(s));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("flag barrier: P=%d CTAs x 512 thr: %.3f us per barrier\n", sms, 1e3f * ms / R);
    }
    {
        unsigned* bar;
        CK(cudaMalloc(&bar, 4096));
        CK(cudaMemset(bar, 0, 4096));
        const int R = 2000;
        for (int v = 0; v < 2; ++v) {
            auto k = v ? split_kernel<32> : split_kernel<0>;
            k<<<sms, 512, 0, s>>>(bar, 10, sink);
            CK(cudaStreamSynchronize(s));
            CK(cudaEventRecord(e0, s));
            k<<<sms, 512, 0, s>>>(bar, R, sink);
            CK(cudaEventRecord(e1, s));
            CK(cudaStreamSynchronize(s));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            printf("split-line barrier (sleep %d): P=%d CTAs x 512 thr: %.3f us per barrier\n", v ? 32 : 0, sms, 1e3f * ms / R);
        }
    }
    for (int pdl = 0; pdl < 2; ++pdl) {
        const int N = 500;
        cudaGraph_t g;
        cudaGraphExec_t ge;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
        for (int i = 0; i < N; ++i) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(sms);
            cfg.blockDim = dim3(512);
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = pdl;
            CK(cudaLaunchKernelEx(&cfg, empty_kernel, sink, pdl));
        }
        CK(cudaStreamEndCapture(s, &g));
        CK(cudaGraphInstantiate(&ge, g, 0));
        CK(cudaGraphLaunch(ge, s));
        CK(cudaStreamSynchronize(s));
        CK(cudaEventRecord(e0, s));
        for (int it = 0; it < 5; ++it) CK(cudaGraphLaunch(ge, s));
        CK(cudaEventRecord(e1, s));
        CK(cudaStreamSynchronize(s));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("kernel boundary (graph, %d CTAs x 512, pdl=%d): %.3f us per kernel\n", sms, pdl, 1e3f * ms / (5 * N));
    }
    return 0;
}
