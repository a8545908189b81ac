// k_viterbi.cu -- tail-biting trellis quantizer on the GPU (PAPER.md:127-141 Viterbi, :331-353
// Algorithm 4), the step that produces the packed streams the GEMV decodes (SURVEY.md 8(f)
// NEXT-1).  L = 16, V = 1, kV in {2, 3}; one CTA (1024 threads) per sequence at a time,
// persistent over the batch.
//
// The DP: V_t(y) = min over the 2^kV predecessors x = c 2^(L-kV) + (y >> kV) of
// V_{t-1}(x), plus (C_y - s_t)^2.  States sharing a group q = y >> kV share their predecessor
// set P(q) = {c 2^(L-kV) + q}, so a step is: m_t(q) = min_{x in P(q)} V_{t-1}(x) for the
// 2^(L-kV) groups, V_t(y) = m_t(y >> kV) + d(y, t).  Ownership follows the de Bruijn structure:
// "base" b in [0, 2^(L-2kV)) owns the groups c 2^(L-2kV) + b (c < 2^kV) and their 2^(2kV)
// states, which are exactly P((b << kV) | j) for j < 2^kV.  So the owner of b turns the minima
// of its own groups (read from shared memory) straight into the next minima of the groups
// (b << kV) | j -- V_t itself is never stored -- and writes those back after a barrier.  Per
// thread: 64 states; per step its 2^kV x (bases per thread) minima in, the same number out,
// 64 x (convert, sub, mul, add, compare).  The code values C_y = fp32(binary16 code(y))
// (bit-exact with qtip_decode) sit in shared memory; the argmins (kV bits per group, one u32
// per thread per step) go to a per-CTA global backpointer array walked back at the end.
//
// Arithmetic is binary32 with every operation rounded on its own (no FMA contraction), in the
// order of the oracle's binary32 DP (oracle/viterbi.c qo_viterbi_f32, reading R17): ties go to
// the smallest predecessor index c and the smallest final state (reading R4).
#include <type_traits>

#include "decode.cuh"
#include "internal.h"

namespace qtip {
namespace {

constexpr int kVThreads = 1024;
constexpr int kVStates = 64;                   // states per thread (2^16 / 1024)

struct ViterbiArgs {
    CodeArgs ca;
    int code;
    const float* src;                          // [nseq][T], in code units
    const uint32_t* lut;                       // HYB: 2^9 words (c0 | c1 << 16)
    int nseq, T;
    uint32_t* states;                          // [nseq][T / V]
    float* cost;                               // [nseq]
    uint32_t* bp;                              // per CTA: [T][kVThreads] words
};

// Group-minimum array layout: q -> q ^ ((q >> 5) & 31).  The writes (q = (b << kV) | j, lanes
// 2^(2kV) floats apart) and the reads (q = c 2^(16-2kV) + tid BPT + bb) both hit 32 distinct banks.
__device__ __forceinline__ int mphys(int q) { return q ^ ((q >> 5) & 31); }

__device__ __forceinline__ __half code_half(uint32_t y, const CodeArgs& ca, int code) {
    if (code == QTIP_CODE_3INST) return inst3_value(inst3_word(y, ca.a, ca.b, ca.magic));
    return onemad_value(onemad_sum(y, ca.a, ca.b));
}

template <int KV>
__global__ void __launch_bounds__(kVThreads, 1) viterbi_kernel(const ViterbiArgs args) {
    constexpr int L = 16;
    constexpr int SH = L - KV;                         // group index bits
    constexpr int NB = 1 << (L - 2 * KV);              // bases
    constexpr int BPT = NB / kVThreads;                // bases per thread (2^(6 - 2kV))
    constexpr int NC = 1 << KV;
    static_assert(BPT * NC * NC == kVStates, "64 states per thread");
    extern __shared__ __align__(16) float sm[];
    float* M = sm;                                     // [2^SH] group minima
    __half* codeh = reinterpret_cast<__half*>(sm + (1 << SH));   // [1024][64] this thread's C_y
    float* s_src = sm + (1 << SH) + kVThreads * kVStates / 2;    // [T] source of the pass
    __shared__ float red_v[32];
    __shared__ uint32_t red_i[32];
    __shared__ uint32_t s_state;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int T = args.T;
    uint32_t* bp = args.bp + (size_t)blockIdx.x * T * kVThreads;
    // slot i = (bb NC + j) NC + c <-> base b = tid BPT + bb, group q = c NB + b, state (q << KV) | j;
    // code halves stored chunk-interleaved (8 halves of a thread per 16-B chunk, chunks of all
    // threads side by side) so a warp's vector loads are conflict-free
    auto state_of = [&](int i) {
        const int bb = i / (NC * NC), j = (i / NC) % NC, c = i % NC;
        return ((uint32_t)(c * NB + tid * BPT + bb) << KV) | (uint32_t)j;
    };
    auto hoff = [&](int i) { return ((i >> 3) * kVThreads + tid) * 8 + (i & 7); };
#pragma unroll 4
    for (int i = 0; i < kVStates; ++i) codeh[hoff(i)] = code_half(state_of(i), args.ca, args.code);
    // the NC code values of (bb, j), c = 0 .. NC-1, as floats
    auto codes_of = [&](int bb, int j, float (&cv)[NC]) {
        const int i0 = (bb * NC + j) * NC;
        if constexpr (NC == 8) {
            const uint4 q = *reinterpret_cast<const uint4*>(codeh + hoff(i0));
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[k]));
                cv[2 * k] = f.x;
                cv[2 * k + 1] = f.y;
            }
        } else {
            const uint2 q = *reinterpret_cast<const uint2*>(codeh + hoff(i0));
            const uint32_t w[2] = {q.x, q.y};
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[k]));
                cv[2 * k] = f.x;
                cv[2 * k + 1] = f.y;
            }
        }
    };

    for (int seq = blockIdx.x; seq < args.nseq; seq += gridDim.x) {
        const float* s = args.src + (size_t)seq * T;
        uint32_t O = 0;
        for (int pass = 0; pass < 2; ++pass) {
            // pass 0: s rotated right by floor(T/2), free ends; pass 1: s, overlap O at both ends
            __syncthreads();
            for (int t = tid; t < T; t += kVThreads) s_src[t] = pass ? s[t] : s[(t - T / 2 + T) % T];
            __syncthreads();
            // m for step 1: the minima over P(q') of V_0, V_0(y) = d(y, 0) (or inf off the start set)
            float m[BPT * NC];                              // this thread's group minima (c, bb)
            // step t: V_{t-1}(y) = m_{t-1}(q(y)) + d(y, t-1) folded into the minima m_t of (b << KV) | j;
            // the first step (V_0 = d, start constraint) is a separate instantiation so the main
            // loop is branch-free
            auto step = [&](int t, auto kFirst) {
                constexpr bool first = decltype(kFirst)::value;
                const float st = s_src[t - 1];
                uint32_t word = 0;
#pragma unroll
                for (int bb = 0; bb < BPT; ++bb)
#pragma unroll
                    for (int j = 0; j < NC; ++j) {
                        float best = INFINITY;
                        uint32_t bc = 0;
                        float cv[NC];
                        codes_of(bb, j, cv);
#pragma unroll
                        for (int c = 0; c < NC; ++c) {
                            const float e = __fsub_rn(cv[c], st);
                            const float d = __fmul_rn(e, e);
                            float x;
                            if constexpr (first) x = (pass == 0 || (uint32_t)(c * NB + tid * BPT + bb) == O) ? d : INFINITY;
                            else x = __fadd_rn(m[c * BPT + bb], d);
                            if (x < best) { best = x; bc = c; }
                        }
                        M[mphys(((tid * BPT + bb) << KV) | j)] = best;
                        word |= bc << ((bb * NC + j) * KV);
                    }
                bp[(size_t)t * kVThreads + tid] = word;
                __syncthreads();
#pragma unroll
                for (int bb = 0; bb < BPT; ++bb)
#pragma unroll
                    for (int c = 0; c < NC; ++c) m[c * BPT + bb] = M[mphys(c * NB + tid * BPT + bb)];
                __syncthreads();                                // M is rewritten by the next step
            };
            if (T > 1) step(1, std::true_type{});
            for (int t = 2; t < T; ++t) step(t, std::false_type{});
            // final state (recomputed V_{T-1}): smallest cost, then smallest index
            float best = INFINITY;
            uint32_t by = 0xFFFFFFFFu;
            {
                const float st = s_src[T - 1];
#pragma unroll
                for (int bb = 0; bb < BPT; ++bb)
#pragma unroll
                    for (int j = 0; j < NC; ++j) {
                        float cv[NC];
                        codes_of(bb, j, cv);
#pragma unroll
                        for (int c = 0; c < NC; ++c) {
                            const uint32_t y = ((uint32_t)(c * NB + tid * BPT + bb) << KV) | (uint32_t)j;
                            const float e = __fsub_rn(cv[c], st);
                            const float d = __fmul_rn(e, e);
                            const float x = T == 1 ? ((pass == 0 || (y >> KV) == O) ? d : INFINITY)
                                                   : __fadd_rn(m[c * BPT + bb], d);
                            const bool ok = pass == 0 || (y & ((1u << SH) - 1u)) == O;
                            if (ok && (x < best || (x == best && y < by))) { best = x; by = y; }
                        }
                    }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const float ob = __shfl_xor_sync(0xffffffffu, best, o);
                const uint32_t oy = __shfl_xor_sync(0xffffffffu, by, o);
                if (ob < best || (ob == best && oy < by)) { best = ob; by = oy; }
            }
            if (lane == 0) { red_v[warp] = best; red_i[warp] = by; }
            __syncthreads();
            if (warp == 0) {
                best = red_v[lane];
                by = red_i[lane];
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    const float ob = __shfl_xor_sync(0xffffffffu, best, o);
                    const uint32_t oy = __shfl_xor_sync(0xffffffffu, by, o);
                    if (ob < best || (ob == best && oy < by)) { best = ob; by = oy; }
                }
                if (lane == 0) {
                    // no finite walk (tail-biting infeasible, kT < L): state 0, as the oracle's strict <
                    if (!(best < INFINITY)) by = 0;
                    // backpointers: group q of y -> base q >> KV (thread (q >> KV) / BPT), slot q & (NC-1)
                    uint32_t y = by;
                    const int g = T / 2;                    // Alg. 4 seam: 1-indexed group floor(T/(2V)) (R3)
                    if (pass == 1) {
                        args.states[(size_t)seq * T + T - 1] = y;
                        args.cost[seq] = best;
                    }
                    if (pass == 0 && g - 1 == T - 1) s_state = y & ((1u << SH) - 1u);
                    for (int t = T - 1; t >= 1; --t) {
                        const uint32_t q = y >> KV;
                        const uint32_t b = q >> KV, jj = q & (NC - 1);
                        const uint32_t w = __ldcg(bp + (size_t)t * kVThreads + b / BPT);
                        const uint32_t c = (w >> (((b % BPT) * NC + jj) * KV)) & (NC - 1);
                        y = (c << SH) | q;
                        if (pass == 1) args.states[(size_t)seq * T + t - 1] = y;
                        if (pass == 0 && t - 1 == g - 1) {
                            s_state = y & ((1u << SH) - 1u);
                            break;
                        }
                    }
                }
            }
            __syncthreads();
            O = s_state;
        }
    }
}


// ---------------------------------------------------------------------------------------------
// V = 2 (HYB): kV = 2k in {4, 6, 8}; a step consumes a pair of source values and the
// state's code is the LUT pair (c0, c1) of h = y^2 + y with the sign of c1 from bit 15 of h (one
// sign).  2^kV predecessors per group are too many to keep a base's states in one thread, so each
// thread holds JT of the base's j and CT of its c (JT CT BPT = 64 states); for kV = 8 four adjacent
// lanes split the c of one j and combine their minima with two shuffles (smaller c wins ties).
// The code is evaluated on the fly from a 2^(Q+1) = 1024-entry table with the sign folded in
// (entries 512..1023 carry -c1), replicated 32-fold in shared memory (index bits 6..15 of h).
// Group minima live in two swapped shared-memory arrays, base-major (position b 2^kV + c) so a
// thread's c run is contiguous; backpointers are one byte per group per step.
// V1 = true: the same de Bruijn ownership for V = 1 codes with kV = 4 (3INST / 1MAD at k = 4): one
// source value per step, the computed code of the state (bit-exact with qtip_decode) instead of the
// HYB pair, d = (C_y - s_t)^2 (reading R17's binary32 order), seam at group floor(T / 2) (R3).
template <int KV, bool V1 = false>
__global__ void __launch_bounds__(kVThreads, 1) viterbi2_kernel(const ViterbiArgs args) {
    constexpr int L = 16;
    constexpr int SH = L - KV;
    constexpr int NB = 1 << (L - 2 * KV);              // bases
    constexpr int NC = 1 << KV;
    constexpr int NG = 1 << SH;                        // groups
    constexpr int TPB = kVThreads / NB;                // threads per base (>= 4 here)
    constexpr int CSPLIT = TPB > NC ? TPB / NC : 1;    // lanes sharing one j (kV = 8: 4)
    constexpr int JT = TPB > NC ? 1 : NC / TPB;        // j per thread
    constexpr int CT = NC / CSPLIT;                    // c per thread
    static_assert(JT * CT == kVStates, "64 states per thread");
    extern __shared__ __align__(16) float sm[];
    float* Mbuf = sm;                                                  // [2][NG], position b NC + c
    uint32_t* lut = reinterpret_cast<uint32_t*>(sm + 2 * NG);          // [1024][32] words (c0 | c1 << 16)
    float* s_src = sm + 2 * NG + 1024 * 32;                            // [T]
    __shared__ float red_v[32];
    __shared__ uint32_t red_i[32];
    __shared__ uint32_t s_state;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int T = args.T, nsteps = V1 ? T : T / 2;
    uint8_t* bp = reinterpret_cast<uint8_t*>(args.bp) + (size_t)blockIdx.x * nsteps * NG;
    const int b = tid / TPB;
    const int jbase = TPB > NC ? (tid % TPB) / CSPLIT : (tid % TPB) * JT;
    const int cbase = TPB > NC ? (tid % CSPLIT) * CT : 0;
    if constexpr (!V1) {
        for (int i = tid; i < 1024 * 32; i += kVThreads) {
            const int e = i >> 5;
            uint32_t w = args.lut[e & 511];
            if (e & 512) w ^= 0x80000000u;                             // c1 negated (Alg. 3 bit 15)
            lut[i] = w;
        }
    }
    const uint32_t lut_lane = (uint32_t)__cvta_generic_to_shared(lut) + 4u * lane;
    auto pos = [](int q) { return (q % NB) * NC + q / NB; };            // base-major group position

    for (int seq = blockIdx.x; seq < args.nseq; seq += gridDim.x) {
        const float* s = args.src + (size_t)seq * T;
        uint32_t O = 0;
        for (int pass = 0; pass < 2; ++pass) {
            __syncthreads();
            for (int t = tid; t < T; t += kVThreads) s_src[t] = pass ? s[t] : s[(t - T / 2 + T) % T];
            __syncthreads();
            int cur = 0;
            // V_{t-1}(y) = m_{t-1}(q(y)) + d(y, t-1) folded into m_t((b << KV) | j)
            auto step = [&](int t, auto kFirst, auto kLast, float& fbest, uint32_t& fy) {
                constexpr bool first = decltype(kFirst)::value, last = decltype(kLast)::value;
                const float s0 = V1 ? s_src[t - 1] : s_src[2 * (t - 1)], s1 = V1 ? 0.0f : s_src[2 * (t - 1) + 1];
                const float* M = Mbuf + cur * NG;
                float* Mn = Mbuf + (cur ^ 1) * NG;
#pragma unroll 1
                for (int jj = 0; jj < JT; ++jj) {
                    const int j = jbase + jj;
                    float best = INFINITY;
                    uint32_t bc = 0;
#pragma unroll 4
                    for (int cc = 0; cc < CT; ++cc) {
                        const int c = cbase + cc;
                        const uint32_t y = ((uint32_t)(c * NB + b) << KV) | (uint32_t)j;
                        float d;
                        if constexpr (V1) {
                            const float e0 = __fsub_rn(__half2float(code_half(y, args.ca, args.code)), s0);
                            d = __fmul_rn(e0, e0);
                        } else {
                            const uint32_t h2 = y * (y + y + 2u);        // 2 (y^2 + y) mod 2^32
                            uint32_t v;
                            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(lut_lane + (h2 & 0x1FF80u)));
                            const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&v));
                            const float e0 = __fsub_rn(f.x, s0), e1 = __fsub_rn(f.y, s1);
                            d = __fadd_rn(__fmul_rn(e0, e0), __fmul_rn(e1, e1));
                        }
                        float x;
                        if constexpr (first) x = (pass == 0 || (uint32_t)(c * NB + b) == O) ? d : INFINITY;
                        else x = __fadd_rn(M[b * NC + c], d);
                        if constexpr (last) {
                            const bool ok = pass == 0 || (y & ((1u << SH) - 1u)) == O;
                            if (ok && (x < fbest || (x == fbest && y < fy))) { fbest = x; fy = y; }
                        } else if (x < best) {
                            best = x;
                            bc = c;
                        }
                    }
                    if constexpr (!last) {
                        if constexpr (CSPLIT > 1) {
#pragma unroll
                            for (int o = 1; o < CSPLIT; o <<= 1) {
                                const float ob = __shfl_xor_sync(0xffffffffu, best, o);
                                const uint32_t oc = __shfl_xor_sync(0xffffffffu, bc, o);
                                if (ob < best || (ob == best && oc < bc)) { best = ob; bc = oc; }
                            }
                        }
                        if (cbase == 0) {
                            const int q = (b << KV) | j;
                            Mn[pos(q)] = best;
                            bp[(size_t)t * NG + q] = (uint8_t)bc;
                        }
                    }
                }
                if constexpr (!last) {
                    __syncthreads();
                    cur ^= 1;
                }
            };
            float fbest = INFINITY;
            uint32_t fy = 0xFFFFFFFFu;
            if (nsteps == 1) {
                step(1, std::true_type{}, std::true_type{}, fbest, fy);
            } else {
                step(1, std::true_type{}, std::false_type{}, fbest, fy);
                for (int t = 2; t < nsteps; ++t) step(t, std::false_type{}, std::false_type{}, fbest, fy);
                step(nsteps, std::false_type{}, std::true_type{}, fbest, fy);
            }
            float best = fbest;
            uint32_t by = fy;
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const float ob = __shfl_xor_sync(0xffffffffu, best, o);
                const uint32_t oy = __shfl_xor_sync(0xffffffffu, by, o);
                if (ob < best || (ob == best && oy < by)) { best = ob; by = oy; }
            }
            if (lane == 0) { red_v[warp] = best; red_i[warp] = by; }
            __syncthreads();
            if (warp == 0) {
                best = red_v[lane];
                by = red_i[lane];
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    const float ob = __shfl_xor_sync(0xffffffffu, best, o);
                    const uint32_t oy = __shfl_xor_sync(0xffffffffu, by, o);
                    if (ob < best || (ob == best && oy < by)) { best = ob; by = oy; }
                }
                if (lane == 0) {
                    if (!(best < INFINITY)) by = 0;
                    uint32_t y = by;
                    // Alg. 4 seam: 1-indexed group floor(T/(2V)) (R3); for T = 2 that is index -1, which the
                    // oracle (Python indexing) reads as the last state
                    const int g = V1 ? T / 2 : T / 4, gi = g >= 1 ? g - 1 : nsteps - 1;
                    if (pass == 1) {
                        args.states[(size_t)seq * nsteps + nsteps - 1] = y;
                        args.cost[seq] = best;
                    }
                    if (pass == 0 && gi == nsteps - 1) s_state = y & ((1u << SH) - 1u);
                    for (int t = nsteps - 1; t >= 1; --t) {
                        const uint32_t q = y >> KV;
                        const uint32_t c = __ldcg(bp + (size_t)t * NG + q);
                        y = (c << SH) | q;
                        if (pass == 1) args.states[(size_t)seq * nsteps + t - 1] = y;
                        if (pass == 0 && t - 1 == gi) {
                            s_state = y & ((1u << SH) - 1u);
                            break;
                        }
                    }
                }
            }
            __syncthreads();
            O = s_state;
        }
    }
}

// the T_x x T_y block (I, J) of W is one sequence, rows concatenated (row-major
// scan); R9: the source enters in code units (multiplied by the code's state standard deviation).
__global__ void gather_sequences_kernel(const float* __restrict__ W, int64_t m, int64_t n, int Tx, int Ty, float scale,
                                        float* __restrict__ out) {
    const int64_t seq = blockIdx.x;
    const int64_t nb = n / Ty;
    const int64_t I = seq / nb, J = seq % nb;
    for (int p = threadIdx.x; p < Tx * Ty; p += blockDim.x)
        out[seq * Tx * Ty + p] = W[(I * Tx + p / Ty) * n + J * Ty + p % Ty] * scale;
}

}  // namespace

cudaError_t launch_gather_sequences(const float* W, int64_t m, int64_t n, int Tx, int Ty, float scale, float* out,
                                    cudaStream_t s) {
    gather_sequences_kernel<<<(unsigned)((m / Tx) * (n / Ty)), 256, 0, s>>>(W, m, n, Tx, Ty, scale, out);
    count_launch(1);
    return cudaGetLastError();
}

size_t viterbi_workspace_bytes(int T) { return (size_t)num_sms() * T * kVThreads * 4; }   // >= V = 2 needs

bool viterbi_supported(int code, int k, int V, int L, int Q, int two_sign) {
    if (L != 16) return false;
    if (code == QTIP_CODE_HYB) return V == 2 && Q == 9 && !two_sign && (k == 2 || k == 3 || k == 4);
    return V == 1 && (k == 2 || k == 3 || k == 4) && (code == QTIP_CODE_3INST || code == QTIP_CODE_1MAD);
}

cudaError_t launch_viterbi(int code, int kv, const CodeArgs& ca, const float* src, const uint16_t* lut, int nseq, int T,
                           uint32_t* states, float* cost, void* ws, cudaStream_t s) {
    ViterbiArgs a;
    a.lut = reinterpret_cast<const uint32_t*>(lut);
    a.ca = ca;
    a.code = code;
    a.src = src;
    a.nseq = nseq;
    a.T = T;
    a.states = states;
    a.cost = cost;
    a.bp = (uint32_t*)ws;
    const int grid = nseq < num_sms() ? nseq : num_sms();
    cudaError_t e = cudaErrorInvalidValue;
    auto go = [&](auto kern, int sh) {
        const size_t smem = ((size_t)1 << sh) * 4 + (size_t)kVThreads * kVStates * 2 + (size_t)T * 4;
        cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (r != cudaSuccess) return r;
        kern<<<grid, kVThreads, smem, s>>>(a);
        return cudaGetLastError();
    };
    auto go2 = [&](auto kern, int sh) {
        const size_t smem = 2 * ((size_t)1 << sh) * 4 + (size_t)1024 * 32 * 4 + (size_t)T * 4;
        cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (r != cudaSuccess) return r;
        kern<<<grid, kVThreads, smem, s>>>(a);
        return cudaGetLastError();
    };
    if (code == QTIP_CODE_HYB) {
        if (kv == 4) e = go2(viterbi2_kernel<4>, 12);
        else if (kv == 6) e = go2(viterbi2_kernel<6>, 10);
        else if (kv == 8) e = go2(viterbi2_kernel<8>, 8);
    } else if (kv == 4) {
        e = go2(viterbi2_kernel<4, true>, 12);
    } else if (kv == 2) e = go(viterbi_kernel<2>, 14);
    else if (kv == 3) e = go(viterbi_kernel<3>, 13);
    count_launch(1);
    return e;
}

}  // namespace qtip
