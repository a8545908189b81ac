// Debug aid: per-SM throughput of integer ops on sm_100a (lanes/clk/SM), 16 warps/SM, 8 independent chains.
#include <cstdio>
#include <cstdint>
#define N_IT 2048
template <int OP>
__global__ void bench(uint32_t* out, long long* cyc, uint32_t s0) {
    uint32_t v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * (i + 3) + s0;
    const uint32_t a = s0 * 7 + 89226354u, b = s0 + 64248484u;
    long long t0 = clock64();
    for (int it = 0; it < N_IT; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) v[i] = v[i] * a + b;                                   // IMAD reg,reg,reg
            if (OP == 1) v[i] = v[i] * 89226354u + 64248484u;                   // IMAD reg,imm (+ reg?)
            if (OP == 2) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(v[i]) : "r"(a));          // IMAD.HI
            if (OP == 3) asm volatile("lop3.b32 %0, %0, %1, %2, 0x6a;" : "+r"(v[i]) : "r"(a), "r"(b));  // LOP3
            if (OP == 4) v[i] = __funnelshift_l(v[i], v[(i + 1) & 7], 5);       // SHF.L.W
            if (OP == 5) asm volatile("prmt.b32 %0, %0, 0, 0x4421;" : "+r"(v[i]));                 // PRMT
            if (OP == 6) v[i] = __dp4a(v[i], 0x01010101u, b);                   // IDP.4A
            if (OP == 7) v[i] = v[i] + b + a;                                   // IADD3
            if (OP == 8) { float f = __uint_as_float(v[i]); f = f * 1.0001f + 0.5f; v[i] = __float_as_uint(f); }  // FFMA imm
        }
    }
    long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc ^= v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    uint32_t* o; long long* c; cudaMalloc(&o, 1 << 24); cudaMalloc(&c, 8);
    const char* names[] = {"IMAD r,r,r", "IMAD r,imm", "IMAD.HI", "LOP3", "SHF.L.W", "PRMT", "IDP.4A", "IADD3", "FFMA imm"};
    auto run = [&](int op, auto kern) {
        for (int warps : {4, 16}) {
            kern<<<1, 32 * warps>>>(o, c, 3);
            long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            double lanes = 32.0 * warps * N_IT * 8;
            printf("%-11s warps=%2d: %.1f lanes/clk/SM  (%.2f cyc per warp-instr per SMSP)\n", names[op], warps, lanes / h,
                   (double)h / (warps / 4.0 * N_IT * 8));
        }
    };
    run(0, bench<0>); run(1, bench<1>); run(2, bench<2>); run(3, bench<3>); run(4, bench<4>);
    run(5, bench<5>); run(6, bench<6>); run(7, bench<7>); run(8, bench<8>);
    return 0;
}
