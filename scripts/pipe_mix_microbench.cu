// pipe_mix_microbench.cu -- do IMAD, LOP3, SHF, PRMT and FFMA issue on separate pipes on sm_100a?
// Each kernel runs 8 independent chains per thread with a fixed mix of two op types; if both ops
// have their own 64-lane pipe the mix reaches 128 lanes/clk/SM, if they share one it stays at 64.
// Decides the decode-loop instruction budget.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_mix_microbench pipe_mix_microbench.cu
#include <cstdint>
#include <cstdio>

#define N_IT 2048

template <int A, int B>
__device__ __forceinline__ uint32_t op(uint32_t x, uint32_t y, uint32_t a, uint32_t b) {
    uint32_t r = x;
    constexpr int O = A;
    (void)B;
    if (O == 0) asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(a), "r"(b));            // IMAD
    if (O == 1) asm volatile("lop3.b32 %0, %1, %2, %3, 0x6a;" : "=r"(r) : "r"(x), "r"(a), "r"(b));        // LOP3
    if (O == 2) asm volatile("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(y), "r"(x), "r"(b));        // SHF
    if (O == 3) asm volatile("prmt.b32 %0, %1, %2, 0x4421;" : "=r"(r) : "r"(x), "r"(y));                   // PRMT
    if (O == 4) {                                                                                           // FFMA
        float f = __uint_as_float(x);
        asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(f) : "f"(f), "f"(__uint_as_float(a)), "f"(__uint_as_float(b)));
        r = __float_as_uint(f);
    }
    if (O == 5) asm volatile("add.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(a));                           // IADD
    return r;
}

// chains 0..3 use op X, chains 4..7 op Y (ratio 1:1); X == Y measures a single type
template <int X, int Y>
__global__ void mix(uint32_t* out, long long* cyc, uint32_t s0) {
    uint32_t v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * (i + 3) + s0;
    const uint32_t a = s0 * 7 + 0x3f800001u, b = s0 + 3u;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < N_IT; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (i & 1) v[i] = op<Y, 0>(v[i], v[(i + 1) & 7], a, b);
            else v[i] = op<X, 0>(v[i], v[(i + 1) & 7], a, b);
        }
    }
    const long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc ^= v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    uint32_t* o;
    long long* c;
    cudaMalloc(&o, 1 << 24);
    cudaMalloc(&c, 8);
    const char* nm[] = {"IMAD", "LOP3", "SHF", "PRMT", "FFMA", "IADD"};
    auto run = [&](int x, int y, auto kern) {
        const int warps = 16;
        kern<<<1, 32 * warps>>>(o, c, 3);
        kern<<<1, 32 * warps>>>(o, c, 3);
        long long h;
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        const double lanes = 32.0 * warps * N_IT * 8;
        printf("%-5s + %-5s: %6.1f lanes/clk/SM\n", nm[x], nm[y], lanes / h);
    };
    run(0, 0, mix<0, 0>);
    run(1, 1, mix<1, 1>);
    run(2, 2, mix<2, 2>);
    run(4, 4, mix<4, 4>);
    run(0, 1, mix<0, 1>);
    run(0, 2, mix<0, 2>);
    run(1, 2, mix<1, 2>);
    run(0, 3, mix<0, 3>);
    run(1, 3, mix<1, 3>);
    run(0, 4, mix<0, 4>);
    run(1, 4, mix<1, 4>);
    run(2, 4, mix<2, 4>);
    run(0, 5, mix<0, 5>);
    run(1, 5, mix<1, 5>);
    return 0;
}
