/* Viterbi dynamic program over an (L, k, V) bitshift trellis -- CPU oracle, TEST INFRASTRUCTURE ONLY.
 *
 * P:129-141 (Sec. 2.3): minimise sum_t ||C_{x_t} - s_t||^2 over walks x_1..x_{T/V}, via
 *   V_t(y) = min_{(x,y) in G} V_{t-1}(x) + ||C_y - s_t||^2 .
 * P:208-209 (Sec. 3.1): x -> y is an edge iff the top L-kV bits of y equal the bottom
 *   L-kV bits of x, so the predecessors of y are x = (c << (L-kV)) | (y >> kV), c < 2^{kV}.
 * P:349 (Alg. 4): "Viterbi(S, G) with start/end overlap = O": the first state's top L-kV
 *   bits and the last state's bottom L-kV bits are both O (a tail-biting walk).
 * Ties (the paper is silent, reading R4): the smallest predecessor index and the smallest
 *   final state win; this equals the reverse-lexicographic minimum among optimal walks.
 * Plain loops, float64, compiled with -ffp-contract=off so sums associate left to right
 * exactly like the Python brute force.  OpenMP only runs independent sequences in parallel.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

static double dist(const double* code, const double* s, int V, uint32_t y, int t) {
    double d = 0.0;
    for (int v = 0; v < V; ++v) {
        double e = code[(size_t)y * V + v] - s[(size_t)t * V + v];
        d += e * e;
    }
    return d;
}

/* overlap < 0: free start and end.  Returns the optimal cost (HUGE_VAL if infeasible, -1 on OOM). */
double qo_viterbi(int L, int kv, int V, int nsteps, const double* code, const double* s, long overlap,
                  uint32_t* out_states) {
    const uint32_t N = 1u << L;
    const int sh = L - kv;
    const uint32_t nc = 1u << kv;
    const uint32_t omask = (sh > 0) ? ((1u << sh) - 1u) : 0u;
    double* cur = (double*)malloc(sizeof(double) * N);
    double* nxt = (double*)malloc(sizeof(double) * N);
    uint8_t* bp = (uint8_t*)malloc((size_t)nsteps * N);
    if (!cur || !nxt || !bp) { free(cur); free(nxt); free(bp); return -1.0; }

    for (uint32_t y = 0; y < N; ++y) {
        int ok = (overlap < 0) || ((y >> kv) == (uint32_t)overlap);
        cur[y] = ok ? dist(code, s, V, y, 0) : HUGE_VAL;
    }
    for (int t = 1; t < nsteps; ++t) {
        for (uint32_t y = 0; y < N; ++y) {
            double best = HUGE_VAL;
            uint32_t bc = 0;
            for (uint32_t c = 0; c < nc; ++c) {
                uint32_t x = (sh > 0 ? (c << sh) : c) | (kv < L ? (y >> kv) : 0u);
                if (cur[x] < best) { best = cur[x]; bc = c; }
            }
            nxt[y] = best + dist(code, s, V, y, t);
            bp[(size_t)t * N + y] = (uint8_t)bc;
        }
        double* tmp = cur; cur = nxt; nxt = tmp;
    }
    double best = HUGE_VAL;
    uint32_t by = 0;
    for (uint32_t y = 0; y < N; ++y) {
        int ok = (overlap < 0) || ((y & omask) == (uint32_t)overlap);
        if (ok && cur[y] < best) { best = cur[y]; by = y; }
    }
    uint32_t y = by;
    out_states[nsteps - 1] = y;
    for (int t = nsteps - 1; t >= 1; --t) {
        uint32_t c = bp[(size_t)t * N + y];
        y = (sh > 0 ? (c << sh) : c) | (kv < L ? (y >> kv) : 0u);
        out_states[t - 1] = y;
    }
    free(cur); free(nxt); free(bp);
    return best;
}

/* Independent sequences S[i*T .. (i+1)*T) with their own overlaps (or -1). */
void qo_viterbi_batch(int L, int kv, int V, int nsteps, const double* code, int nseq, const double* S,
                      const long* overlaps, uint32_t* out_states, double* out_cost) {
    #pragma omp parallel for schedule(dynamic, 1)
    for (int i = 0; i < nseq; ++i) {
        out_cost[i] = qo_viterbi(L, kv, V, nsteps, code, S + (size_t)i * nsteps * V, overlaps[i],
                                 out_states + (size_t)i * nsteps);
    }
}

/* binary32 variant (reading R17): the same DP, every operation a single IEEE binary32
 * operation in the same order -- e = c_y - s_t (sub), e*e (mul), d += (add, V terms left to right),
 * best + d (add), strict < with the smallest index winning.  The GPU quantizer (qtip_viterbi)
 * takes its argmin decisions in binary32, so this is the precision its paths are checked in. */
static float dist_f(const float* code, const float* s, int V, uint32_t y, int t) {
    float d = 0.0f;
    for (int v = 0; v < V; ++v) {
        float e = code[(size_t)y * V + v] - s[(size_t)t * V + v];
        float e2 = e * e;
        d = d + e2;
    }
    return d;
}

float qo_viterbi_f32(int L, int kv, int V, int nsteps, const float* code, const float* s, long overlap,
                     uint32_t* out_states) {
    const uint32_t N = 1u << L;
    const int sh = L - kv;
    const uint32_t nc = 1u << kv;
    const uint32_t omask = (sh > 0) ? ((1u << sh) - 1u) : 0u;
    float* cur = (float*)malloc(sizeof(float) * N);
    float* nxt = (float*)malloc(sizeof(float) * N);
    uint8_t* bp = (uint8_t*)malloc((size_t)nsteps * N);
    if (!cur || !nxt || !bp) { free(cur); free(nxt); free(bp); return -1.0f; }
    for (uint32_t y = 0; y < N; ++y) {
        int ok = (overlap < 0) || ((y >> kv) == (uint32_t)overlap);
        cur[y] = ok ? dist_f(code, s, V, y, 0) : HUGE_VALF;
    }
    for (int t = 1; t < nsteps; ++t) {
        for (uint32_t y = 0; y < N; ++y) {
            float best = HUGE_VALF;
            uint32_t bc = 0;
            for (uint32_t c = 0; c < nc; ++c) {
                uint32_t x = (sh > 0 ? (c << sh) : c) | (kv < L ? (y >> kv) : 0u);
                if (cur[x] < best) { best = cur[x]; bc = c; }
            }
            nxt[y] = best + dist_f(code, s, V, y, t);
            bp[(size_t)t * N + y] = (uint8_t)bc;
        }
        float* tmp = cur; cur = nxt; nxt = tmp;
    }
    float best = HUGE_VALF;
    uint32_t by = 0;
    for (uint32_t y = 0; y < N; ++y) {
        int ok = (overlap < 0) || ((y & omask) == (uint32_t)overlap);
        if (ok && cur[y] < best) { best = cur[y]; by = y; }
    }
    uint32_t y = by;
    out_states[nsteps - 1] = y;
    for (int t = nsteps - 1; t >= 1; --t) {
        uint32_t c = bp[(size_t)t * N + y];
        y = (sh > 0 ? (c << sh) : c) | (kv < L ? (y >> kv) : 0u);
        out_states[t - 1] = y;
    }
    free(cur); free(nxt); free(bp);
    return best;
}

void qo_viterbi_f32_batch(int L, int kv, int V, int nsteps, const float* code, int nseq, const float* S,
                          const long* overlaps, uint32_t* out_states, float* out_cost) {
    #pragma omp parallel for schedule(dynamic, 1)
    for (int i = 0; i < nseq; ++i) {
        out_cost[i] = qo_viterbi_f32(L, kv, V, nsteps, code, S + (size_t)i * nsteps * V, overlaps[i],
                                     out_states + (size_t)i * nsteps);
    }
}
