// k_chain.cu -- impl 8: a chain of dependent QTIP layers in ONE persistent tcgen05 launch.
//
//   stage 0:  y_l = scale_l S_m H_m^T W~_l H_n S_n x                (every layer l)
//   stage s:  the same with x := y_src(s), src(s) a layer of stage s-1
//
// A decode step of a model is such a chain (q,k,v -> o -> gate,up -> down -> next block's q,k,v).
// Per layer the GEMV itself only needs x~ at MMA time: the packed weights (the
// only large traffic) and their trellis decode (Alg. 1-3) do not depend on the activations.  So a
// single grid, one CTA per SM, streams and decodes the weights of ALL layers back to back -- the
// producer and the decoders run ahead of the data into the next layers -- and only the MMAs wait
// for each stage's x~.  The per-layer kernel boundaries of the separate RHT-in -> GEMV -> RHT-out
// kernels (a PDL release after a full grid costs ~1.3 us) disappear; what is left
// per stage transition is a flag hand-off and the transforms, overlapped with the next stage's
// decode.
//
// Roles (18 warps, 576 threads):
//   warp 0      producer: cp.async.bulk of every cell of the CTA's ranges of all stages into an
//               S-stage ring (L2 evict-first).  Never waits on data.
//   warp 1      MMA issuer: per stage waits for the x~ of the layers its range touches (xready
//               counters in global memory), bulk-loads that x~ window into shared memory (double
//               buffered by stage parity), then issues 8 tcgen05.mma (M = 128, N = 16, K = 16, A =
//               decoded weights in TMEM, B = x~ in shared memory) per cell, as in k_umma.cu.
//   warps 2-5   epilogue + transforms: D (TMEM) -> y~ rows or stream-K segments of split row
//               blocks (last arriver adds them in range order), a done counter per layer; then
//               this CTA's share of the stage transition's transforms:
//                 Tout(l): y_l = scale S_m (H_m^T y~_l)/sqrt(m)   (user output, fp32)
//                 Tin(l'): x~_l' = H_n (S_n y_src)/sqrt(n)         (binary16, UMMA B layout)
//               each task waits on a counter (done / yready) and bumps one (yready / xready).
//   warps 6-17  three decoder groups (thread = TMEM lane = row of a cell), udec::decode_pair.
//
// Transforms (reading R7: H_n = H_b (x) H_{2^a}).  With L2 = 2^a2 (a2 = a for a <= 5, 5 if 5 < a < 7,
// else min(a, 12)) and the dense factor D = H_b (x) H_{2^(a-a2)} of order f = n / L2,
//     (H v)[i L2 + c] = FWHT_L2( sum_j D[i][j] V[j][.] )[c],     V[j][c] = v[j L2 + c],
// so a task owns R rows i of D and needs every V[j] once (read from L2) and no other task's
// result.  L2 <= 32: lane c of an L2-lane group accumulates its rows and the FWHT runs in
// shuffles; L2 >= 128: thread = column (mod 128), the lowest 5 FWHT levels in shuffles, the rest in
// radix-8 passes over shared memory.  The inverse uses D^T (H_b^T: Paley-I is skew, reading R8).
//
// Deadlock freedom (every CTA resident: cooperative launch): each role walks the stages in order;
// weights and decode never wait on data; a CTA's epilogue warps do E(s-1) then the transition-s
// tasks (all Tout before all Tin on every CTA), Tout waits only on E(s-1) of all CTAs, Tin only on
// Tout.  Shared-memory reuse: the x~ buffer of stage s-2 is the transition-s scratch... see the
// barrier notes in the kernel.
#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.h"
#include "umma_decode.cuh"

namespace qtip {
namespace {

constexpr int kCG = 2;                        // decoder groups
constexpr int kCWarps = 10 + 4 * kCG;         // producer, MMA, 4 epilogue, 4 transform, decoders
constexpr int kCThreads = 32 * kCWarps;       // 576
constexpr int kCNBuf = 3;                     // TMEM A buffers per decoder group
constexpr int kXfBar = 2;                     // named barrier of the transform warps
constexpr uint32_t kCHdr = 1024;
constexpr uint32_t kCLutQ = 9;
constexpr uint32_t kCLutBytes = (1u << (kCLutQ + 1)) * 128u;
constexpr int kMaxStageLayers = 4;
constexpr int kXfThreads = 128;               // the epilogue warps

struct Xform {
    int n;          // transform length (m for the inverse, n for the forward)
    int b, a1;      // D = H_b (x) H_{2^a1}
    int L2;         // FWHT length done per row
    int f;          // order of D (= b 2^a1), n = f L2
    int R;          // rows of D per task
    int ntask;
};

struct ChainLayerDev {
    const uint32_t* packed;
    const uint8_t* sign_n;
    const uint8_t* sign_m;
    const uint32_t* hb_n;      // H_b bit rows for the forward over n (nullptr if b = 1)
    const uint32_t* hbt_m;     // H_b^T bit rows for the inverse over m (nullptr if b = 1)
    float* y;                  // user output [B][m]
    uint16_t* xt;              // x~ [n_pad / 8][BP][8] binary16 (RHT out_mode 7)
    float* yt;                 // y~ [B][m_pad]
    float* seg;                // stream-K segments [(P + n_rb)][BP][128]
    int* ticket;               // [n_rb] arrivals (zero between launches)
    float scale;
    int m, n, n_rb, n_kc;
    int src;                   // execution index of the layer whose y is the input (-1: the external x)
    int rd0, rd1;              // readers: layers [rd0, rd1) (execution order) take this layer's y as input
    int U;                     // cells (n_rb n_kc)
    Xform out, in;
};

struct ChainArgs {
    const ChainLayerDev* L;    // in execution order
    int nlayers;
    int* ctr;                  // done[nl] | yready[nl] | xready[nl]
    const float* x;            // external input [B][n of stage 0]
    const uint32_t* lut;       // HYB: 2^Q words (c0 | c1 << 16), shared by the chain
    CodeArgs ca;
    int B, BP;
    uint32_t xcol_bytes, lbo, sbo;
    uint32_t off_ring, off_x, xbuf_bytes, off_scr;
};

__host__ __device__ constexpr int chain_stages(int K, int code) { return code == QTIP_CODE_HYB ? 6 : (K == 2 ? 12 : 8); }

__device__ __forceinline__ int range_lo(int U, int W, int w) { return (int)((uint32_t)U * (uint32_t)w / (uint32_t)W); }
__device__ __forceinline__ int range_of(int U, int W, int u) {
    return (int)((((uint32_t)u + 1u) * (uint32_t)W - 1u) / (uint32_t)U);
}
// Debug progress words (qtip_internal_set_chain_debug; null in normal operation): 8 ints per CTA,
// written as each role advances (host-mapped memory, read by scripts/chain_debug.py while it runs).
__device__ int* g_chain_dbg = nullptr;
__device__ int g_chain_yield = 1;        // decoders pause while a transform task runs (knob)
#define CDBG(slot, val)                                           \
    do {                                                          \
        if (dbg) *(volatile int*)(dbg + (slot)) = (int)(val);     \
    } while (0)

// Debug timeline (qtip_internal_set_chain_trace; null in normal operation): %globaltimer ns at
// [(cta * kTrStages + stage) * 8 + event], stages < kTrStages.  Events: 0 MMA starts waiting for the
// stage's x~, 1 window landed, 2 last MMA issued, 3 epilogue E(stage) done, 4 first transition task
// of T(stage+1) starts, 5 T(stage+1) done, 6 decoders' first cell of the stage, 7 producer's first cell.
constexpr int kTrStages = 160;
__device__ unsigned long long* g_chain_trace = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define CTR(stage, ev)                                                                          \
    do {                                                                                        \
        if (trc && (stage) < kTrStages) trc[((size_t)cta * kTrStages + (stage)) * 8 + (ev)] = gtimer(); \
    } while (0)

// A stage of U cells is cut into W = min(P, U) non-empty ranges; CTA w < W runs range w.
__device__ __forceinline__ int stage_ranges(int U, int P) { return U < P ? U : P; }
__device__ __forceinline__ void cta_range(int U, int P, int cta, int& ua, int& ub) {
    const int W = stage_ranges(U, P);
    ua = cta < W ? range_lo(U, W, cta) : 0;
    ub = cta < W ? range_lo(U, W, cta + 1) : 0;
}
__device__ __forceinline__ void warp_arrive(uint32_t bar, int lane) {
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(bar);
}
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void spin_until(const int* p, int target) {
    while (ld_acquire(p) < target) __nanosleep(32);
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// D[i][j] of a transform (sign as +-1.0f): H_b[i_b][j_b] (-1)^popcount(i_1 & j_1), i = i_b 2^a1 + i_1;
// hrow = the H_b bit row of i_b (staged in shared memory).
__device__ __forceinline__ float dsign(const uint32_t* hrow, int b, int a1, int i, int j) {
    const int jb = j >> a1, m1 = (1 << a1) - 1;
    uint32_t s = __popc((uint32_t)(i & j & m1)) & 1u;
    if (b > 1) s ^= (hrow[jb >> 5] >> (jb & 31)) & 1u;
    return s ? -1.0f : 1.0f;
}
// Stage the H_b bit rows of D rows r0 .. r0+R-1 into hbits[rl * wpr + w] (wpr = ceil(b / 32)).
__device__ __forceinline__ void stage_hbits(const uint32_t* __restrict__ hb, const Xform& X, int r0, int R,
                                            uint32_t* hbits, int tid) {
    if (X.b <= 1) return;
    const int wpr = (X.b + 31) >> 5;
    for (int e = tid; e < R * wpr; e += kXfThreads) hbits[e] = __ldg(hb + (size_t)((r0 + e / wpr) >> X.a1) * wpr + e % wpr);
}

// Scratch layout of a transform task (floats): [ssg: sign bytes n/8][ssg2: the fused source's S_m]
// [D: L2 <= 32: D^(T) rows as [f][8] floats; L2 >= 128: f floats (one row)][buf: reduction / exchange].
__host__ __device__ inline int xf_sign_floats(int n) { return ((n / 8 + 15) & ~15) / 4; }
__host__ __device__ inline int xf_d_floats(const Xform& X) {           // D (+ the staged H_b bit rows)
    return (X.L2 <= 32 ? 8 * X.f : ((X.f + 3) & ~3)) + ((8 * ((X.b + 31) >> 5) + 3) & ~3);
}
__host__ __device__ inline int xf_buf_floats(const Xform& X) {
    return X.L2 <= 32 ? 8 * 128 : X.L2 + X.L2 / 32;   // small: [slots][R <= 8][L2] partial sums; large: the row (zp)
}

// Where a task's results go (kept in registers: the layer descriptor itself is a local copy).
struct XfOut {
    uint16_t* xt;      // dir 0: x~ (binary16, UMMA B layout, batch pad BP)
    float* y;          // dir 1: y [B][m]
    int m, BP, dir;
};
// Output element e of batch row bt: x~ or y (S_m applied; the scale is in v).
__device__ __forceinline__ void xf_store(const XfOut& o, int bt, int e, float v, const uint8_t* sgn) {
    if (o.dir == 0) {
        o.xt[(e >> 3) * 8 * o.BP + 8 * bt + (e & 7)] = __half_as_ushort(__float2half_rn(v));
    } else {
        o.y[(int64_t)bt * o.m + e] = ((sgn[e >> 3] >> (e & 7)) & 1u) ? -v : v;
    }
}
__device__ __forceinline__ float sgnf(const uint8_t* s, int e, float v) { return ((s[e >> 3] >> (e & 7)) & 1u) ? -v : v; }

// Copy nbytes (even) of sign bytes to shared memory with every load of a batch in flight at once
// (a loop of load -> store would pay one L2 round trip per iteration).
__device__ __forceinline__ void stage_signs(uint8_t* dst, const uint8_t* __restrict__ src, int nbytes, int tid) {
    const uint16_t* s16 = reinterpret_cast<const uint16_t*>(src);
    uint16_t* d16 = reinterpret_cast<uint16_t*>(dst);
    const int nh = nbytes >> 1;
    for (int b0 = 0; b0 < nh; b0 += 8 * kXfThreads) {
        uint16_t t[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int e = b0 + tid + kXfThreads * i;
            t[i] = e < nh ? __ldg(s16 + e) : (uint16_t)0;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int e = b0 + tid + kXfThreads * i;
            if (e < nh) d16[e] = t[i];
        }
    }
}

// L2 >= 128 transforms work in shared memory with compact loops and no register arrays: with the
// kernel's 227 KB shared-memory carve-out the L1 data cache is ~29 KB, so a register-heavy FWHT that
// spills to local memory pays an L2 round trip per spill (ncu: long-scoreboard stalls on the
// butterflies), and unrolled code runs cold out of the instruction cache at each transition.
// Element e of a row lives at float zp(e) = e + 4 (e / 128) (16-byte aligned float4 runs; radix-8
// passes with h >= 64 are conflict-free, h = 1, 8 at most 4-way).
__device__ __forceinline__ int zp(int e) { return e + 4 * (e >> 7); }

// In-place FWHT of length L2 (pow2 >= 128) on Z, radix-8 / 4 / 2 passes over 128 threads; two
// groups per thread per iteration so their shared-memory loads overlap.
__device__ void fwht_smem(float* Z, int L2, int tid) {
    for (int h = 1; h < L2;) {
        const int rem = L2 / h;
        const int lv = rem >= 8 ? 3 : rem >= 4 ? 2 : 1;
        const int r = 1 << lv, ng = L2 >> lv;
        ptx::named_bar_sync(kXfBar, kXfThreads);
#pragma unroll 1
        for (int g0 = tid; g0 < ng; g0 += 2 * kXfThreads) {
            float v[2][8];
            int base[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int g = g0 + u * kXfThreads;
                base[u] = (g / h) * (h * r) + (g % h);
                if (g < ng) {
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        if (k < r) v[u][k] = Z[zp(base[u] + k * h)];
                }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
#pragma unroll
                for (int hh = 1; hh < 8; hh <<= 1)
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        if (hh < r && !(k & hh) && k + hh < r) {
                            const float p0 = v[u][k], p1 = v[u][k + hh];
                            v[u][k] = p0 + p1;
                            v[u][k + hh] = p0 - p1;
                        }
                if (g0 + u * kXfThreads < ng) {
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        if (k < r) Z[zp(base[u] + k * h)] = v[u][k];
                }
            }
        }
        h <<= lv;
    }
    ptx::named_bar_sync(kXfBar, kXfThreads);
}

// L2 >= 128, one row (r0) of D per task: Z = sum_j D[r0][j] X[j][.] (input signs applied), FWHT_L2,
// store.  Fused (Ls != nullptr, pow2 n, f = 1): X is first y_src computed here from the source's y~
// (inverse FWHT, scale_src S_m,src / sqrt(n)), so the task needs no hand-off.
__device__ void xf_large(const XfOut& o, const ChainLayerDev& Ld, const ChainLayerDev* Ls, int dir, int bt,
                         const float* inb, const Xform& X, int r0, const uint32_t* hb, uint8_t* ssg, uint8_t* ssg2,
                         float* Dsm, float* Z, float fac, int tid, unsigned long long* tt) {
    const int f = X.f, L2 = X.L2, n = X.n;
    const int nq = L2 / 4;                               // float4 runs per row
    const uint8_t* sg = dir ? Ld.sign_m : Ld.sign_n;
    // every load of the row (float4, coalesced) in flight at once, then into shared memory
    if (f == 1) {                                        // cp.async: no registers, all in flight
        for (int q = tid; q < nq; q += kXfThreads)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ptx::smem_u32(Z + zp(4 * q))),
                         "l"(reinterpret_cast<const float4*>(inb) + q)
                         : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    stage_signs(ssg, sg, n / 8, tid);
    if (Ls) stage_signs(ssg2, Ls->sign_m, n / 8, tid);
    uint32_t* hbits = reinterpret_cast<uint32_t*>(Dsm + ((f + 3) & ~3));
    stage_hbits(hb, X, r0, 1, hbits, tid);
    if (f == 1) asm volatile("cp.async.wait_group 0;" ::: "memory");
    ptx::named_bar_sync(kXfBar, kXfThreads);
    for (int e = tid; e < f; e += kXfThreads) Dsm[e] = dsign(hbits, X.b, X.a1, r0, e);
    ptx::named_bar_sync(kXfBar, kXfThreads);
    if (tt && tid == 0) tt[1] = gtimer();
    if (Ls) {
        // y_src = scale_src S_m,src (H^T y~_src) / sqrt(n); the forward's input is S_n y_src
        fwht_smem(Z, L2, tid);
        const float fs = Ls->scale * rsqrtf((float)n);
#pragma unroll 4
        for (int e = tid; e < L2; e += kXfThreads) Z[zp(e)] = sgnf(ssg, e, sgnf(ssg2, e, Z[zp(e)] * fs));
    } else if (f == 1) {
        const float d0 = Dsm[0];
        if (dir == 0 || d0 != 1.0f) {
#pragma unroll 4
            for (int e = tid; e < L2; e += kXfThreads) Z[zp(e)] = (dir == 0 ? sgnf(ssg, e, Z[zp(e)]) : Z[zp(e)]) * d0;
        }
    } else {
        // Z[c] = sum_j D[j] X[j][c]; thread: float4 runs q of the row, rows j in batches of 4
#pragma unroll 1
        for (int q = tid; q < nq; q += kXfThreads) {
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
            for (int j0 = 0; j0 < f; j0 += 4) {
                float4 x[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (j0 + i < f) x[i] = __ldcg(reinterpret_cast<const float4*>(inb + (j0 + i) * L2) + q);
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (j0 + i < f) {
                        const int e = (j0 + i) * L2 + 4 * q;
                        const float d = Dsm[j0 + i];
                        float4 xv = x[i];
                        if (dir == 0) {
                            xv.x = sgnf(ssg, e, xv.x);
                            xv.y = sgnf(ssg, e + 1, xv.y);
                            xv.z = sgnf(ssg, e + 2, xv.z);
                            xv.w = sgnf(ssg, e + 3, xv.w);
                        }
                        acc.x = fmaf(d, xv.x, acc.x);
                        acc.y = fmaf(d, xv.y, acc.y);
                        acc.z = fmaf(d, xv.z, acc.z);
                        acc.w = fmaf(d, xv.w, acc.w);
                    }
            }
            *reinterpret_cast<float4*>(Z + zp(4 * q)) = acc;
        }
    }
    if (tt && tid == 0) tt[2] = gtimer();
    fwht_smem(Z, L2, tid);
    if (tt && tid == 0) tt[3] = gtimer();
#pragma unroll 2
    for (int q = tid; q < nq; q += kXfThreads) {
        const float4 w = *reinterpret_cast<const float4*>(Z + zp(4 * q));
        const int e = r0 * L2 + 4 * q;
        if (o.dir == 0 && o.BP == 1) {
            const __half2 h01 = __floats2half2_rn(w.x * fac, w.y * fac), h23 = __floats2half2_rn(w.z * fac, w.w * fac);
            uint2 u;
            u.x = *reinterpret_cast<const uint32_t*>(&h01);
            u.y = *reinterpret_cast<const uint32_t*>(&h23);
            *reinterpret_cast<uint2*>(o.xt + e) = u;
        } else if (o.dir == 1) {
            float4 y;
            y.x = sgnf(ssg, e, w.x * fac);
            y.y = sgnf(ssg, e + 1, w.y * fac);
            y.z = sgnf(ssg, e + 2, w.z * fac);
            y.w = sgnf(ssg, e + 3, w.w * fac);
            *reinterpret_cast<float4*>(o.y + (int64_t)bt * o.m + e) = y;
        } else {
            xf_store(o, bt, e, w.x * fac, ssg);
            xf_store(o, bt, e + 1, w.y * fac, ssg);
            xf_store(o, bt, e + 2, w.z * fac, ssg);
            xf_store(o, bt, e + 3, w.w * fac, ssg);
        }
    }
    if (tt && tid == 0) tt[4] = gtimer();
    ptx::named_bar_sync(kXfBar, kXfThreads);            // Z / signs are reused by the next batch row
}

// L2 <= 32: R <= 8 rows of D per task.  Thread (jslot, c): c = column, the j-slot takes rows j = slot,
// slot + nslot, ... of X (a warp reads 32 consecutive floats per j), accumulates all R rows (D^T row
// j of 8 floats, broadcast), in register batches of 32 loads; the slots' partial sums are added in
// slot order through shared memory, then FWHT_L2 across the lanes and the store.
__device__ void xf_small(const XfOut& o, const ChainLayerDev& Ld, int dir, int bt, const float* inb, const Xform& X,
                         int r0, int R, const uint32_t* hb, uint8_t* ssg, float* Dt, float* red, float fac, int tid,
                         unsigned long long* tt) {
    const int lane = tid & 31, f = X.f, L2 = X.L2, n = X.n;
    const uint8_t* sg = dir ? Ld.sign_m : Ld.sign_n;
    const int c = lane & (L2 - 1);
    const int nslot = kXfThreads / L2, slot = tid / L2;
    const int nj = (f - slot + nslot - 1) / nslot;       // this thread's rows of X
    constexpr int JB = 8;
    float xa[JB], xb[JB];
    auto load = [&](float (&xv)[JB], int i0) {
#pragma unroll
        for (int i = 0; i < JB; ++i) xv[i] = i0 + i < nj ? __ldcg(inb + (slot + nslot * (i0 + i)) * L2 + c) : 0.0f;
    };
    load(xa, 0);
    stage_signs(ssg, sg, n / 8, tid);
    uint32_t* hbits = reinterpret_cast<uint32_t*>(Dt + 8 * f);
    stage_hbits(hb, X, r0, R, hbits, tid);
    ptx::named_bar_sync(kXfBar, kXfThreads);
    const int wpr = (X.b + 31) >> 5;
    for (int e = tid; e < 8 * f; e += kXfThreads) {
        const int j = e >> 3, rl = e & 7;
        Dt[e] = rl < R ? dsign(hbits + rl * wpr, X.b, X.a1, r0 + rl, j) : 0.0f;
    }
    ptx::named_bar_sync(kXfBar, kXfThreads);
    if (tt && tid == 0) tt[1] = gtimer();
    float acc[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) acc[r] = 0.0f;
    auto consume = [&](const float (&xv)[JB], int i0) {
#pragma unroll
        for (int i = 0; i < JB; ++i) {
            if (i0 + i >= nj) break;
            const int j = slot + nslot * (i0 + i);
            const float x = dir == 0 ? sgnf(ssg, j * L2 + c, xv[i]) : xv[i];
            const float4 d0 = *reinterpret_cast<const float4*>(Dt + 8 * j);
            const float4 d1 = *reinterpret_cast<const float4*>(Dt + 8 * j + 4);
            acc[0] = fmaf(d0.x, x, acc[0]);
            acc[1] = fmaf(d0.y, x, acc[1]);
            acc[2] = fmaf(d0.z, x, acc[2]);
            acc[3] = fmaf(d0.w, x, acc[3]);
            acc[4] = fmaf(d1.x, x, acc[4]);
            acc[5] = fmaf(d1.y, x, acc[5]);
            acc[6] = fmaf(d1.z, x, acc[6]);
            acc[7] = fmaf(d1.w, x, acc[7]);
        }
    };
    // two register batches in flight: load batch i+1 while consuming batch i
    for (int i0 = 0; i0 < nj; i0 += 2 * JB) {
        if (i0 + JB < nj) load(xb, i0 + JB);
        consume(xa, i0);
        if (i0 + 2 * JB < nj) load(xa, i0 + 2 * JB);
        if (i0 + JB < nj) consume(xb, i0 + JB);
    }
    if (tt && tid == 0) tt[2] = gtimer();
    // partial sums [slot][r][c] -> Z[r][c] = sum over slots in slot order
#pragma unroll
    for (int r = 0; r < 8; ++r)
        if (r < R) red[(slot * 8 + r) * L2 + c] = acc[r];
    ptx::named_bar_sync(kXfBar, kXfThreads);
    for (int o0 = 0; o0 < 8 * L2; o0 += kXfThreads) {
        const int r = (o0 + tid) / L2;
        float z = 0.0f;
        if (r < R)
            for (int sl = 0; sl < nslot; ++sl) z += red[(sl * 8 + r) * L2 + c];
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
            if (s >= L2) break;
            const float oz = __shfl_xor_sync(0xffffffffu, z, s);
            z = (lane & s) ? oz - z : z + oz;
        }
        if (r < R) xf_store(o, bt, (r0 + r) * L2 + c, z * fac, ssg);
    }
    if (tt && tid == 0) tt[3] = tt[4] = gtimer();
    ptx::named_bar_sync(kXfBar, kXfThreads);                  // red / signs are reused by the next batch row
}

// One transform task on the 128 epilogue threads (tid 0..127, named barrier 1).  dir 0: x~ of
// layer Ld from its input (fused: from the source's y~); dir 1: y of layer Ld from its y~.
// sm: scratch (the idle x~ buffer).  Every global read of a phase is issued before its first use
// (the inputs live in L2: a chain of dependent L2 round trips, not bandwidth, is what a 16-44 KB
// transform would otherwise cost).
__device__ void run_xform(const ChainArgs& a, const ChainLayerDev& Ld, const ChainLayerDev* Ls, int dir, int part,
                          float* sm, int tid, unsigned long long* tt = nullptr) {
    if (tt && tid == 0) tt[0] = gtimer();
    const Xform X = dir ? Ld.out : Ld.in;
    const int n = X.n;
    const int r0 = part * X.R, R = min(X.R, X.f - r0);
    const float* in;
    int64_t in_stride;
    if (Ls) {
        in = Ls->yt;
        in_stride = (int64_t)Ls->n_rb * 128;
    } else if (dir == 0) {
        in = Ld.src < 0 ? a.x : a.L[Ld.src].y;
        in_stride = n;
    } else {
        in = Ld.yt;
        in_stride = (int64_t)Ld.n_rb * 128;
    }
    const uint32_t* hb = dir ? Ld.hbt_m : Ld.hb_n;
    const float fac = dir ? Ld.scale * rsqrtf((float)n) : rsqrtf((float)n);
    uint8_t* ssg = reinterpret_cast<uint8_t*>(sm);
    uint8_t* ssg2 = reinterpret_cast<uint8_t*>(sm + xf_sign_floats(n));
    float* Dsm = sm + 2 * xf_sign_floats(n);
    float* buf = Dsm + xf_d_floats(X);
    XfOut o;
    o.xt = Ld.xt;
    o.y = Ld.y;
    o.m = Ld.m;
    o.BP = a.BP;
    o.dir = dir;
    for (int bt = 0; bt < a.B; ++bt) {
        const float* inb = in + bt * in_stride;
        if (X.L2 <= 32) {
            xf_small(o, Ld, dir, bt, inb, X, r0, R, hb, ssg, Dsm, buf, fac, tid, tt);
        } else {
            xf_large(o, Ld, Ls, dir, bt, inb, X, r0, hb, ssg, ssg2, Dsm, buf, fac, tid, tt);
        }
    }
    if (tt && tid == 0) tt[5] = gtimer();
}

// Is layer Ld's x~ computed by one fused task straight from its source's y~ (power-of-two n, one task
// each way)?  Then it waits for the source's done counter, not for the source's y.
__device__ __forceinline__ bool xf_fused(const ChainLayerDev& Ld, const ChainLayerDev* L) {
    return Ld.src >= 0 && Ld.in.f == 1 && Ld.in.L2 >= 128 && L[Ld.src].out.f == 1 && L[Ld.src].out.L2 >= 128;
}

template <int K, int CODE, bool kImm>
__global__ void __launch_bounds__(kCThreads, 1) chain_kernel(const __grid_constant__ ChainArgs a) {
    constexpr bool kHyb = CODE == QTIP_CODE_HYB;
    constexpr int S = chain_stages(K, CODE);
    constexpr int N = 16;
    constexpr uint32_t kCellBytes = 2048u * K;
    constexpr int kTW = 8 * K;
    constexpr uint32_t kACols = 64;
    constexpr uint32_t kD1 = N;
    constexpr uint32_t kA0 = 128;
    static_assert(kA0 + kCG * kCNBuf * kACols <= 512, "TMEM budget");
    constexpr uint32_t idesc = ptx::idesc_f16_f32(128, N);

    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    const uint32_t bar0 = ptx::smem_u32(smem);
    auto full = [&](int s) { return bar0 + 8u * s; };
    auto empty = [&](int s) { return bar0 + 8u * (S + s); };
    auto afull = [&](int g, int b) { return bar0 + 8u * (2 * S + g * kCNBuf + b); };
    auto aempty = [&](int g, int b) { return bar0 + 8u * (2 * S + kCG * kCNBuf + g * kCNBuf + b); };
    const uint32_t barD = bar0 + 8u * (2 * S + 2 * kCG * kCNBuf);
    auto dfull = [&](int d) { return barD + 8u * d; };
    auto dempty = [&](int d) { return barD + 16u + 8u * d; };
    auto xfull = [&](int b) { return barD + 32u + 8u * b; };      // x~ window b landed
    auto xfree = [&](int b) { return barD + 48u + 8u * b; };      // MMAs reading window b done
    // a transform task is running on this CTA's epilogue warps: the decoders yield the issue slots
    volatile int* s_xbusy = reinterpret_cast<volatile int*>(smem + 1004);
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + 1016);
    uint8_t* ring = smem + a.off_ring;
    const int P = (int)gridDim.x;
    const int cta = (int)blockIdx.x;
    const int nl = a.nlayers;
    const ChainLayerDev* __restrict__ Lg = a.L;
    int* const dbg = g_chain_dbg ? g_chain_dbg + 8 * cta : nullptr;
    unsigned long long* const trc = g_chain_trace;

    if constexpr (kHyb) {
        uint4* lt = reinterpret_cast<uint4*>(smem + kCHdr);
        for (int i = threadIdx.x; i < (1 << (kCLutQ + 1)) * 8; i += kCThreads) {
            const int e = i >> 3;
            uint32_t w = __ldg(a.lut + (e & ((1 << kCLutQ) - 1)));
            if (e >> kCLutQ) w ^= 0x80000000u;
            lt[i] = make_uint4(w, w, w, w);
        }
    }
    if (warp == 0) {
        if (lane == 0) {
            for (int s = 0; s < S; ++s) {
                ptx::mbar_init(full(s), 1);
                ptx::mbar_init(empty(s), 4);
            }
            for (int g = 0; g < kCG; ++g)
                for (int b = 0; b < kCNBuf; ++b) {
                    ptx::mbar_init(afull(g, b), 4);
                    ptx::mbar_init(aempty(g, b), 1);
                }
            for (int d = 0; d < 2; ++d) {
                ptx::mbar_init(dfull(d), 1);
                ptx::mbar_init(dempty(d), 4);
                ptx::mbar_init(xfull(d), 1);
                ptx::mbar_init(xfree(d), 1);
            }
            ptx::fence_mbar_init();
            *s_xbusy = 0;
        }
        __syncwarp();
        ptx::tmem_alloc(ptx::smem_u32(tmem_holder), 512);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_holder, 0);

    // Sub-stage l = layer l (execution order: stage by stage, the next stage's source first): its
    // U cells in W = min(P, U) equal ranges, CTA w < W runs range w.
    if (warp == 0) {
        // ================= producer: every cell of this CTA's range of every layer, in order
        const uint64_t pol = ptx::l2_evict_first_policy();
        int s = 0;
        uint32_t r = 0;
        bool wrapped = false;
        const int64_t cw = kCellBytes / 4;                // words per cell
        for (int l = 0; l < nl; ++l) {
            int ua, ub;
            cta_range(Lg[l].U, P, cta, ua, ub);
            if (ua >= ub) continue;
            if (lane == 0) CTR(l, 7);
            const uint32_t* src = Lg[l].packed + (int64_t)ua * cw;
            for (int u = ua; u < ub; ++u) {
                if (wrapped) ptx::mbar_wait_sleep(empty(s), r ^ 1u);
                if (ptx::elect_one()) {
                    ptx::mbar_arrive_expect_tx(full(s), kCellBytes);
                    ptx::bulk_g2s_policy(ptx::smem_u32(ring + (size_t)s * kCellBytes), src, kCellBytes, full(s), pol);
                }
                __syncwarp();
                if (lane == 0) CDBG(0, u + 1000000 * l);
                if (++s == S) { s = 0; r ^= 1u; wrapped = true; }
                src += cw;
            }
        }
    } else if (warp == 1) {
        // ================= x~ window loader + MMA issuer
        int seg = 0, jj = 0;
        const uint32_t dstep = 2u * (uint32_t)a.BP;
        for (int l = 0; l < nl; ++l) {
            const ChainLayerDev& Ld = Lg[l];
            const int nkc = Ld.n_kc;
            int ua, ub;
            cta_range(Ld.U, P, cta, ua, ub);
            const int xb = l & 1;
            const uint32_t xwin = ptx::smem_u32(smem + a.off_x + (uint32_t)xb * a.xbuf_bytes);
            if (lane == 0) CDBG(1, 10 * l + 2);
            if (l >= 2) ptx::mbar_wait_sleep(xfree(xb), (uint32_t)(((l - 2) >> 1) & 1));   // window b's MMAs of layer l-2
            // the window: columns of the range's cells (all n_kc when it covers a whole row block)
            const int cnt = ub - ua < nkc ? ub - ua : nkc;
            const int kcs = ub - ua < nkc ? ua % nkc : 0;
            if (lane == 0) {
                if (ua < ub) {
                    CTR(l, 0);
                    spin_until(a.ctr + 2 * nl + l, Ld.in.ntask);
                    fence_proxy_async_global();
                    ptx::fence_proxy_async_smem();
                    ptx::mbar_arrive_expect_tx(xfull(xb), (uint32_t)cnt * a.xcol_bytes);
                    const uint8_t* xs = reinterpret_cast<const uint8_t*>(Ld.xt);
                    const int run1 = cnt < nkc - kcs ? cnt : nkc - kcs;
                    ptx::bulk_g2s(xwin, xs + (size_t)kcs * a.xcol_bytes, (uint32_t)run1 * a.xcol_bytes, xfull(xb));
                    if (cnt > run1)
                        ptx::bulk_g2s(xwin + (uint32_t)run1 * a.xcol_bytes, xs, (uint32_t)(cnt - run1) * a.xcol_bytes,
                                      xfull(xb));
                } else {
                    ptx::mbar_arrive(xfull(xb));            // keep the window barrier's phases aligned
                }
            }
            __syncwarp();
            ptx::mbar_wait_sleep(xfull(xb), (uint32_t)((l >> 1) & 1));
            if (lane == 0 && ua < ub) CTR(l, 1);
            ptx::tc_fence_after();
            if (ua < ub) {
                int KC = ua % nkc;
                int off = (KC - kcs + nkc) % nkc;
                uint32_t dcol = tmem;
                bool first = true;
                for (int u = ua; u < ub; ++u, ++jj) {
                    if (u == ua || KC == 0) {
                        const int d = seg & 1;
                        if (seg >= 2) ptx::mbar_wait_sleep(dempty(d), (uint32_t)(((seg >> 1) - 1) & 1));
                        ptx::tc_fence_after();
                        dcol = tmem + (uint32_t)d * kD1;
                        first = true;
                    }
                    const int g = jj % kCG, lc = jj / kCG, b = lc % kCNBuf;
                    ptx::mbar_wait_sleep(afull(g, b), (uint32_t)((lc / kCNBuf) & 1));
                    if (lane == 0) CDBG(2, jj);
                    ptx::tc_fence_after();
                    const uint64_t cdesc = ptx::smem_desc_kmajor_noswizzle(xwin + (uint32_t)off * a.xcol_bytes, a.lbo, a.sbo);
                    const uint32_t acol = tmem + kA0 + (uint32_t)(g * kCNBuf + b) * kACols;
                    const bool seg_end = (u + 1 == ub) || (KC == nkc - 1);
                    if (ptx::elect_one()) {
#pragma unroll
                        for (int i = 0; i < 8; ++i)
                            ptx::umma_f16_ts(dcol, acol + 8u * (uint32_t)i, cdesc + (uint64_t)(dstep * (uint32_t)i), idesc,
                                             (first && i == 0) ? 0u : 1u);
                        ptx::umma_commit(aempty(g, b));
                        if (seg_end) ptx::umma_commit(dfull(seg & 1));
                    }
                    __syncwarp();
                    first = false;
                    if (seg_end) ++seg;
                    if (++off == nkc) off = 0;
                    if (++KC == nkc) KC = 0;
                }
            }
            if (lane == 0) CTR(l, 2);
            if (ptx::elect_one()) ptx::umma_commit(xfree(xb));   // this layer's MMAs read window xb
            __syncwarp();
        }
    } else if (warp < 6) {
        // ================= epilogue E(l): D -> y~ rows / stream-K segments, the done counters
        __shared__ int s_last;
        const int q = warp & 3;
        const int R = 32 * q + lane;                  // TMEM lane = row of the row block
        const int tid = (int)threadIdx.x - 64;        // 0..127 over warps 2-5
        const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16);
        int seg = 0;
        for (int l = 0; l < nl; ++l) {
            const ChainLayerDev& Lr = Lg[l];
            int ua, ub;
            cta_range(Lr.U, P, cta, ua, ub);
            const int W = stage_ranges(Lr.U, P);
            const int nkc = Lr.n_kc;
            float* const yt = Lr.yt;
            const int mp = Lr.n_rb * 128;
            for (int RB = ua < ub ? ua / nkc : 1, RBe = ua < ub ? (ub - 1) / nkc : 0; RB <= RBe; ++RB, ++seg) {
                const int d = seg & 1;
                if (tid == 0) CDBG(3, 100 * l + 1);
                const int w0 = range_of(Lr.U, W, RB * nkc), w1 = range_of(Lr.U, W, (RB + 1) * nkc - 1);
                const bool whole = w0 == w1;
                float* segp = Lr.seg + ((int64_t)(w0 + RB) * a.BP) * 128 + R;
                float* dst = segp + (int64_t)(cta - w0) * a.BP * 128;
                ptx::mbar_wait_sleep(dfull(d), (uint32_t)((seg >> 1) & 1));
                ptx::tc_fence_after();
                uint32_t rr[16];
                ptx::tmem_ld16(tl + (uint32_t)d * kD1, rr);
                ptx::tc_wait_ld();
                ptx::tc_fence_before();
                warp_arrive(dempty(d), lane);
#pragma unroll
                for (int bb = 0; bb < 16; ++bb) {
                    if (bb >= a.B) break;
                    const float v = __uint_as_float(rr[bb]);
                    if (whole) yt[(int64_t)bb * mp + RB * 128 + R] = v;
                    else dst[bb * 128] = v;
                }
                bool fin = whole;
                if (!whole) {
                    __threadfence();
                    ptx::named_bar_sync(1, kXfThreads);
                    if (tid == 0) {
                        const int old = atomicAdd(Lr.ticket + RB, 1);
                        const bool last = old == w1 - w0;
                        if (last) Lr.ticket[RB] = 0;
                        s_last = last ? 1 : 0;
                    }
                    ptx::named_bar_sync(1, kXfThreads);
                    fin = s_last != 0;
                    if (fin) {
                        __threadfence();
                        const int cnt = w1 - w0 + 1;
                        for (int bb = 0; bb < a.B; ++bb) {
                            const float* sp = segp + bb * 128;
                            float acc = __ldcg(sp);
                            for (int j = 1; j < cnt; ++j) acc += __ldcg(sp + (int64_t)j * a.BP * 128);
                            yt[(int64_t)bb * mp + RB * 128 + R] = acc;
                        }
                    }
                }
                if (fin) {
                    // the row block of y~ is final: count it (release)
                    ptx::named_bar_sync(1, kXfThreads);
                    if (tid == 0) {
                        __threadfence();
                        atomicAdd(a.ctr + l, 1);
                    }
                }
            }
            if (tid == 0) CTR(l, 3);
        }
    } else if (warp < 10) {
        // ================= transforms T(l): Tout(l), then Tin(r) of every reader r of l (l = -1: Tin
        // of the layers reading x); task j of T(l) on CTA (j + 7 (l + 1)) mod P; every CTA runs all
        // Tout of T(l) before its Tin, and T(l) before T(l+1)
        const int tid = (int)threadIdx.x - 192;       // 0..127 over warps 6-9
        float* scratch = reinterpret_cast<float*>(smem + a.off_scr);
        for (int l = -1; l < nl; ++l) {
            int nto = 0, rd0, rd1;
            if (l >= 0) {
                nto = Lg[l].out.ntask;
                rd0 = Lg[l].rd0;
                rd1 = Lg[l].rd1;
            } else {
                rd0 = 0;
                rd1 = 0;
                while (rd1 < nl && Lg[rd1].src < 0) ++rd1;
            }
            int nti = 0;
            for (int r = rd0; r < rd1; ++r) nti += Lg[r].in.ntask;
            const int rot = (int)((7ll * (l + 1)) % P);
            int j = cta - rot;
            if (j < 0) j += P;
            if (l >= 0 && tid == 0 && j < nto + nti) CTR(l, 4);
            for (; j < nto + nti; j += P) {
                const int dir = j < nto ? 1 : 0;
                int jr = j, li = l;
                if (!dir) {
                    jr = j - nto;
                    li = rd0;
                    while (jr >= Lg[li].in.ntask) jr -= Lg[li++].in.ntask;
                }
                const ChainLayerDev& Ld = Lg[li];
                const bool fused = !dir && xf_fused(Ld, Lg);
                if (tid == 0) {
                    if (dir) spin_until(a.ctr + li, Ld.n_rb);
                    else if (fused) spin_until(a.ctr + Ld.src, Lg[Ld.src].n_rb);
                    else if (Ld.src >= 0) spin_until(a.ctr + nl + Ld.src, Lg[Ld.src].out.ntask);
                    *s_xbusy = g_chain_yield;
                }
                ptx::named_bar_sync(kXfBar, kXfThreads);
                unsigned long long* tt = (trc && l >= 0 && l < kTrStages)
                    ? trc + (size_t)P * kTrStages * 8 + ((size_t)cta * kTrStages + l) * 8 : nullptr;
                run_xform(a, Ld, fused ? Lg + Ld.src : nullptr, dir, jr, scratch, tid, tt);
                if (!dir) fence_proxy_async_global();
                __threadfence();
                if (tt && tid == 0) tt[6] = gtimer();
                ptx::named_bar_sync(kXfBar, kXfThreads);
                if (tid == 0) {
                    *s_xbusy = 0;
                    atomicAdd(a.ctr + (dir ? nl : 2 * nl) + li, 1);
                }
            }
            if (l >= 0 && tid == 0) CTR(l, 5);
        }
    } else {
        // ================= decoders: cells jj = g, g + kCG, ... of the CTA's cell sequence
        const int dw = warp - 10, g = dw >> 2, q = warp & 3;
        const int R = 32 * q + lane, I = R >> 4, rho = R & 15;
        const uint32_t ta_lane = tmem + ((uint32_t)(32 * q) << 16) + kA0;
        const uint32_t lut_lane = ptx::smem_u32(smem + kCHdr) + 4u * (uint32_t)lane;
        int ncell = 0;
        for (int l = 0; l < nl; ++l) {
            int ua, ub;
            cta_range(Lg[l].U, P, cta, ua, ub);
            ncell += ub - ua;
        }
        int lc = 0;
        for (int jj = g; jj < ncell; jj += kCG, ++lc) {
            const int s = jj % S;
            const uint32_t r = (uint32_t)((jj / S) & 1);
            const int b = lc % kCNBuf, use = lc / kCNBuf;
            while (*s_xbusy) __nanosleep(64);
            ptx::mbar_wait_sleep(full(s), r);
            if (use > 0) ptx::mbar_wait_sleep(aempty(g, b), (uint32_t)((use - 1) & 1));
            ptx::tc_fence_after();
            const uint32_t* cellw = reinterpret_cast<const uint32_t*>(ring + (size_t)s * kCellBytes);
            const uint32_t ta = ta_lane + (uint32_t)(g * kCNBuf + b) * kACols;
#pragma unroll 1
            for (int pp = 0; pp < 4; ++pp)
                udec::decode_pair<K, CODE, kImm>(cellw + (I * 4 + pp) * kTW * 2, rho, a.ca, lut_lane, ta + (uint32_t)pp * 16);
            warp_arrive(empty(s), lane);
            ptx::tc_wait_st();
            ptx::tc_fence_before();
            warp_arrive(afull(g, b), lane);
            if (lane == 0 && q == 0) CDBG(5 + g, jj);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

// Debug: one transform task alone (1 CTA, the 128 transform threads), timed with clock64.
__global__ void __launch_bounds__(kXfThreads, 1) xform_bench_kernel(const __grid_constant__ ChainArgs a, int li, int dir,
                                                                  int part, int fused, int iters,
                                                                  unsigned long long* out) {
    extern __shared__ __align__(16) uint8_t smx[];
    const int tid = threadIdx.x;
    const ChainLayerDev& Ld = a.L[li];
    const ChainLayerDev* Ls = fused ? a.L + Ld.src : nullptr;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) run_xform(a, Ld, Ls, dir, part, reinterpret_cast<float*>(smx), tid);
    __syncthreads();
    if (tid == 0) out[0] = clock64() - t0;
}

template <int K, int CODE, bool kImm>
cudaError_t launch_chain_t(const ChainArgs& a, int P, size_t smem, cudaStream_t s) {
    auto kern = chain_kernel<K, CODE, kImm>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    prefer_max_smem((const void*)kern);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)P);
    cfg.blockDim = dim3(kCThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

// Transform geometry over length n (reading R7): see the file comment.  L2 <= 32: rows of D per task
// so that a transform has about min(64, P/2) tasks; L2 >= 128: one row of D per task (L2 <= 4096,
// and <= 2048 when D is not trivial, so the row's columns fit 32 registers per thread).
bool make_xform(int64_t n, int P, Xform* X) {
    int b = 0, a = 0;
    if (!hadamard_factor(n, &b, &a)) return false;
    int a2 = a <= 5 ? a : (a < 7 ? 5 : std::min(a, 12));
    X->n = (int)n;
    X->b = b;
    X->a1 = a - a2;
    X->L2 = 1 << a2;
    X->f = (int)(n >> a2);
    const int target = std::max(1, std::min(64, P / 2));
    X->R = X->L2 >= 128 ? 1 : std::min(8, std::max(1, (X->f + target - 1) / target));
    X->ntask = (X->f + X->R - 1) / X->R;
    return true;
}

size_t xform_scratch_bytes(const Xform& X) {
    return 4 * ((size_t)2 * xf_sign_floats(X.n) + xf_d_floats(X) + xf_buf_floats(X));
}

}  // namespace
}  // namespace qtip

// ------------------------------------------------------------------------------------ C ABI
using namespace qtip;

struct qtip_chain_plan {
    std::vector<void*> xt, yt;     // per-layer internal buffers (debug readout)
    int device = 0;
    int code = 0, k = 0;
    bool imm = false;
    int P = 0;
    int nstages = 0, nlayers = 0;
    int64_t B = 0;
    size_t smem = 0;
    ChainArgs args{};
    void* dmem = nullptr;          // one allocation: tables, counters, per-layer buffers
    size_t ctr_bytes = 0;
    int* ctr = nullptr;
};

extern "C" {

qtip_status qtip_chain_plan_create(const qtip_params* p, int32_t nlayers, const qtip_chain_layer* layers, int64_t B,
                                   const uint16_t* d_lut, qtip_chain_plan** out) {
    if (!out) return api_fail(QTIP_ERR_INVALID_PARAMS, "plan pointer is NULL");
    *out = nullptr;
    qtip_status st = qtip_params_check(p);
    if (st != QTIP_OK) return st;
    if (nlayers < 1 || !layers) return api_fail(QTIP_ERR_INVALID_PARAMS, "need at least one layer");
    if (B < 1 || B > 16) return api_fail(QTIP_ERR_UNSUPPORTED, "chain kernel: batch must be in 1..16");
    if (p->k < 2 || p->k > 4) return api_fail(QTIP_ERR_UNSUPPORTED, "chain kernel: needs 2 <= k <= 4");
    if (p->code == QTIP_CODE_HYB && (p->Q != (int)kCLutQ || p->hyb_two_sign || !d_lut))
        return api_fail(QTIP_ERR_UNSUPPORTED, "chain kernel: HYB needs Q = 9, one-sign, and a LUT");
    const int P = num_sms();
    const int BP = B <= 1 ? 1 : B <= 2 ? 2 : B <= 4 ? 4 : B <= 8 ? 8 : 16;
    // ---- validate the layer list (user order) and find the stages
    std::vector<int> stage_first;                      // first user index of every stage
    for (int i = 0; i < nlayers; ++i) {
        const qtip_chain_layer& c = layers[i];
        if (!c.d_packed || !c.d_sign_n || !c.d_sign_m || !c.d_y) return api_fail(QTIP_ERR_INVALID_PARAMS, "NULL layer buffer");
        if ((reinterpret_cast<uintptr_t>(c.d_packed) & 15u)) return api_fail(QTIP_ERR_ALIGNMENT, "d_packed must be 16-B aligned");
        if (c.m <= 0 || c.n <= 0 || c.m % kTile || c.n % kTile) return api_fail(QTIP_ERR_SHAPE, "m and n must be positive multiples of 16");
        const int want_stage = i == 0 ? 0 : (c.stage == layers[i - 1].stage ? layers[i - 1].stage : layers[i - 1].stage + 1);
        if (c.stage != want_stage) return api_fail(QTIP_ERR_INVALID_PARAMS, "stages must be numbered 0, 1, ... in layer order");
        if (c.stage == 0 && c.src != -1) return api_fail(QTIP_ERR_INVALID_PARAMS, "stage 0 layers read the external x (src = -1)");
        if (c.stage > 0) {
            if (c.src < 0 || c.src >= i || layers[c.src].stage != c.stage - 1)
                return api_fail(QTIP_ERR_INVALID_PARAMS, "src must be a layer of the previous stage");
            if (layers[c.src].m != c.n) return api_fail(QTIP_ERR_SHAPE, "src layer's m must equal this layer's n");
        }
        if (i > 0 && c.stage == layers[i - 1].stage && (c.n != layers[i - 1].n || c.src != layers[i - 1].src))
            return api_fail(QTIP_ERR_INVALID_PARAMS, "layers of a stage share n and src (one input)");
        if (c.stage >= (int)stage_first.size()) stage_first.push_back(i);
        if (i + 1 - stage_first.back() > kMaxStageLayers)
            return api_fail(QTIP_ERR_UNSUPPORTED, "chain kernel: at most 4 layers per stage");
        int b = 0, a = 0;
        if (!hadamard_factor(c.m, &b, &a) || !hadamard_factor(c.n, &b, &a))
            return api_fail(QTIP_ERR_SHAPE, "no supported Hadamard order for m or n");
    }
    const int nst = (int)stage_first.size();
    stage_first.push_back(nlayers);
    // ---- execution order: stage by stage; within a stage the next stage's source first, so its
    //      transforms overlap the stage's other layers
    std::vector<int> exec, pos(nlayers);
    for (int s = 0; s < nst; ++s) {
        const int src_next = s + 1 < nst ? layers[stage_first[s + 1]].src : -1;
        if (src_next >= 0) exec.push_back(src_next);
        for (int i = stage_first[s]; i < stage_first[s + 1]; ++i)
            if (i != src_next) exec.push_back(i);
    }
    for (int e = 0; e < nlayers; ++e) pos[exec[e]] = e;
    std::vector<ChainLayerDev> L(nlayers);
    for (int e = 0; e < nlayers; ++e) {
        const qtip_chain_layer& c = layers[exec[e]];
        const Layout l = make_layout(c.m, c.n, p->k);
        ChainLayerDev& d = L[e];
        d = ChainLayerDev{};
        d.packed = (const uint32_t*)c.d_packed;
        d.sign_n = c.d_sign_n;
        d.sign_m = c.d_sign_m;
        d.y = c.d_y;
        d.scale = c.scale * (p->code == QTIP_CODE_1MAD ? 5.0f / 739.0f : 1.0f);   // 1MAD: 1/147.8 (reading R6)
        d.m = (int)c.m;
        d.n = (int)c.n;
        d.n_rb = (int)l.n_rb;
        d.n_kc = (int)l.n_kc;
        d.U = d.n_rb * d.n_kc;
        d.src = c.src < 0 ? -1 : pos[c.src];
        d.rd0 = d.rd1 = 0;
        make_xform(c.m, P, &d.out);
        make_xform(c.n, P, &d.in);
        if ((int64_t)d.U * (P + 1) >= (1ll << 31)) return api_fail(QTIP_ERR_UNSUPPORTED, "chain kernel: layer too large");
    }
    for (int s = 0; s + 1 < nst; ++s) {                  // readers of the next stage's source
        const int src = pos[layers[stage_first[s + 1]].src];
        L[src].rd0 = pos[stage_first[s + 1]] < pos[stage_first[s + 1]] ? 0 : nlayers;
        int lo = nlayers, hi = 0;
        for (int i = stage_first[s + 1]; i < stage_first[s + 2]; ++i) {
            lo = std::min(lo, pos[i]);
            hi = std::max(hi, pos[i] + 1);
        }
        L[src].rd0 = lo;
        L[src].rd1 = hi;
    }
    // ---- shared memory: LUT + ring + two x~ windows + the transform scratch
    const bool hyb = p->code == QTIP_CODE_HYB;
    const uint32_t xcol = 128u * 2u * (uint32_t)BP;
    size_t xbuf = 0, scr = 0;
    for (auto& d : L) {
        const int W = std::min(P, d.U);
        const int64_t cw = (d.U + W - 1) / W;
        xbuf = std::max(xbuf, (size_t)std::min<int64_t>(cw, d.n_kc) * xcol);
        scr = std::max({scr, xform_scratch_bytes(d.out), xform_scratch_bytes(d.in)});
    }
    xbuf = (xbuf + 1023) & ~size_t(1023);
    scr = (scr + 1023) & ~size_t(1023);
    const size_t cell = 2048u * (size_t)p->k;
    const size_t lutb = hyb ? kCLutBytes : 0;
    const int S = chain_stages(p->k, p->code);
    const size_t smem = kCHdr + lutb + (size_t)S * cell + 2 * xbuf + scr;
    if (smem > 227 * 1024) return api_fail(QTIP_ERR_UNSUPPORTED, "chain kernel: x~ windows / transform scratch do not fit shared memory");
    // ---- device memory: [layer table][counters + tickets][x~][y~][segments]
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return api_cuda_fail(e, "qtip_chain_plan_create");
    auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
    size_t off = 0;
    const size_t o_L = off; off += al(sizeof(ChainLayerDev) * nlayers);
    const size_t o_ctr = off;
    size_t nctr = 3 * (size_t)nlayers;
    for (auto& d : L) nctr += d.n_rb;
    const size_t ctr_bytes = al(nctr * sizeof(int));
    off += ctr_bytes;
    std::vector<size_t> o_xt(nlayers), o_yt(nlayers), o_seg(nlayers);
    for (int i = 0; i < nlayers; ++i) {
        const ChainLayerDev& d = L[i];
        o_xt[i] = off; off += al((size_t)d.n_kc * 128 * BP * 2);
        o_yt[i] = off; off += al((size_t)B * d.n_rb * 128 * 4);
        o_seg[i] = off; off += al((size_t)(P + d.n_rb) * BP * 128 * 4);
    }
    void* dmem = nullptr;
    if ((e = cudaMalloc(&dmem, off)) != cudaSuccess) return api_cuda_fail(e, "qtip_chain_plan_create: cudaMalloc");
    if ((e = cudaMemset(dmem, 0, off)) != cudaSuccess) {
        cudaFree(dmem);
        return api_cuda_fail(e, "qtip_chain_plan_create: cudaMemset");
    }
    char* base = (char*)dmem;
    int* tk = (int*)(base + o_ctr) + 3 * nlayers;
    for (int i = 0; i < nlayers; ++i) {
        ChainLayerDev& d = L[i];
        d.xt = (uint16_t*)(base + o_xt[i]);
        d.yt = (float*)(base + o_yt[i]);
        d.seg = (float*)(base + o_seg[i]);
        d.ticket = tk;
        tk += d.n_rb;
        d.hb_n = d.in.b > 1 ? hadamard_table_device(d.in.b, false, &e) : nullptr;
        if (e == cudaSuccess) d.hbt_m = d.out.b > 1 ? hadamard_table_device(d.out.b, true, &e) : nullptr;
        if (e != cudaSuccess) {
            cudaFree(dmem);
            return api_cuda_fail(e, "qtip_chain_plan_create: Hadamard tables");
        }
    }
    if ((e = cudaMemcpy(base + o_L, L.data(), sizeof(ChainLayerDev) * nlayers, cudaMemcpyHostToDevice)) != cudaSuccess) {
        cudaFree(dmem);
        return api_cuda_fail(e, "qtip_chain_plan_create: tables");
    }
    qtip_chain_plan* pl = new qtip_chain_plan();
    pl->xt.assign(nlayers, nullptr);
    pl->yt.assign(nlayers, nullptr);
    for (int i = 0; i < nlayers; ++i) {                  // debug readout in the caller's layer order
        pl->xt[exec[i]] = L[i].xt;
        pl->yt[exec[i]] = L[i].yt;
    }
    pl->device = dev;
    pl->code = p->code;
    pl->k = p->k;
    const CodeArgs ca = api_code_args(p);
    pl->imm = !hyb && p->k == 2 && ca.a == (p->code == QTIP_CODE_1MAD ? 34038481u : 89226354u) &&
              ca.b == (p->code == QTIP_CODE_1MAD ? 76625530u : 64248484u);
    pl->P = P;
    pl->nstages = nst;
    pl->nlayers = nlayers;
    pl->B = B;
    pl->smem = smem;
    pl->dmem = dmem;
    pl->ctr = (int*)(base + o_ctr);
    pl->ctr_bytes = ctr_bytes;
    ChainArgs& a = pl->args;
    a.L = (const ChainLayerDev*)(base + o_L);
    a.nlayers = nlayers;
    a.ctr = pl->ctr;
    a.lut = (const uint32_t*)d_lut;
    a.ca = ca;
    a.B = (int)B;
    a.BP = BP;
    a.xcol_bytes = xcol;
    a.lbo = 16u * (uint32_t)BP;
    a.sbo = 128u;
    a.off_ring = (uint32_t)(kCHdr + lutb);
    a.off_x = (uint32_t)(kCHdr + lutb + (size_t)S * cell);
    a.xbuf_bytes = (uint32_t)xbuf;
    a.off_scr = (uint32_t)(a.off_x + 2 * xbuf);
    *out = pl;
    return QTIP_OK;
}

qtip_status qtip_chain_run(qtip_chain_plan* pl, const float* d_x, void* stream) {
    if (!pl || !d_x) return api_fail(QTIP_ERR_INVALID_PARAMS, "NULL plan or x");
    if (reinterpret_cast<uintptr_t>(d_x) & 15u) return api_fail(QTIP_ERR_ALIGNMENT, "d_x must be 16-B aligned");
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(pl->ctr, 0, pl->ctr_bytes, s);
    if (e != cudaSuccess) return api_cuda_fail(e, "qtip_chain_run: counters");
    ChainArgs a = pl->args;
    a.x = d_x;
    e = cudaErrorInvalidValue;
#define QTIP_C_CASE(KK, CC, II) \
    if (pl->k == KK && pl->code == CC && pl->imm == II) e = launch_chain_t<KK, CC, II>(a, pl->P, pl->smem, s);
    QTIP_C_CASE(2, QTIP_CODE_3INST, true) QTIP_C_CASE(2, QTIP_CODE_1MAD, true)
    QTIP_C_CASE(2, QTIP_CODE_3INST, false) QTIP_C_CASE(2, QTIP_CODE_1MAD, false)
    QTIP_C_CASE(3, QTIP_CODE_3INST, false) QTIP_C_CASE(3, QTIP_CODE_1MAD, false)
    QTIP_C_CASE(4, QTIP_CODE_3INST, false) QTIP_C_CASE(4, QTIP_CODE_1MAD, false)
    QTIP_C_CASE(2, QTIP_CODE_HYB, false) QTIP_C_CASE(3, QTIP_CODE_HYB, false) QTIP_C_CASE(4, QTIP_CODE_HYB, false)
#undef QTIP_C_CASE
    count_launch(1);
    if (e != cudaSuccess) return api_cuda_fail(e, "qtip_chain_run: launch");
    return QTIP_OK;
}

void qtip_chain_plan_destroy(qtip_chain_plan* pl) {
    if (!pl) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(pl->device);
    cudaFree(pl->dmem);
    cudaSetDevice(cur);
    delete pl;
}

int32_t qtip_chain_plan_stages(const qtip_chain_plan* pl) { return pl ? pl->nstages : 0; }

}  // extern "C"

extern "C" int qtip_internal_chain_buffers(qtip_chain_plan* pl, int i, void** xt, void** yt) {
    if (!pl || i < 0 || i >= pl->nlayers) return -1;
    *xt = pl->xt[i];
    *yt = pl->yt[i];
    return 0;
}

extern "C" int qtip_internal_chain_xform_bench(qtip_chain_plan* pl, int li, int dir, int part, int fused, int iters,
                                               void* d_out, void* d_x) {
    ChainArgs a = pl->args;
    a.x = (const float*)d_x;
    cudaFuncSetAttribute(xform_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    xform_bench_kernel<<<1, kXfThreads, 64 * 1024>>>(a, li, dir, part, fused, iters, (unsigned long long*)d_out);
    return (int)cudaDeviceSynchronize();
}

extern "C" int qtip_internal_set_chain_yield(int v) {
    return (int)cudaMemcpyToSymbol(qtip::g_chain_yield, &v, sizeof(v));
}

extern "C" int qtip_internal_set_chain_trace(void* p) {
    unsigned long long* q = (unsigned long long*)p;
    return (int)cudaMemcpyToSymbol(qtip::g_chain_trace, &q, sizeof(q));
}

extern "C" int qtip_internal_set_chain_debug(void* p) {
    int* q = (int*)p;
    return (int)cudaMemcpyToSymbol(qtip::g_chain_dbg, &q, sizeof(q));
}

extern "C" int qtip_internal_copy(void* dst, const void* src, size_t bytes) {
    return (int)cudaMemcpy(dst, src, bytes, cudaMemcpyDefault);
}
