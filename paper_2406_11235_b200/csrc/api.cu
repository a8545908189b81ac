// api.cu -- the extern "C" boundary of libqtip (declared in include/qtip.h).
//
// Host-side validation, the private device layout (common.cuh) and kernel dispatch.  No
// call allocates device memory except the per-device Hadamard table cache (hadamard.cpp).
#include <cmath>
#include <cstring>
#include <string>
#include <mutex>
#include <thread>
#include <unordered_set>
#include <vector>

#include "internal.h"

namespace qtip {
namespace {
thread_local std::string g_err;
thread_local uint64_t g_launches = 0;
thread_local cudaEvent_t g_prof_start = nullptr, g_prof_stop = nullptr;
int g_impl = 0;

qtip_status fail(qtip_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

qtip_status cuda_fail(cudaError_t e, const char* where) {
    g_err = std::string(where) + ": " + cudaGetErrorString(e);
    return QTIP_ERR_CUDA;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// m, n multiples of the block (16 x 16, or T_x x T_y for the LUT code)
qtip_status check_block(const qtip_params* p, int64_t m, int64_t n) {
    if (m % p->Tx || n % p->Ty) return fail(QTIP_ERR_SHAPE, "m, n must be multiples of T_x, T_y");
    return QTIP_OK;
}

CodeArgs code_args(const qtip_params* p) {
    CodeArgs c;
    c.a = p->lcg_a;
    c.b = p->lcg_b;
    c.magic = (p->m_fp16 << 16) | (p->m_fp16 & 0xFFFFu);
    c.Q = p->Q;
    c.two_sign = p->hyb_two_sign;
    return c;
}

qtip_status check_shape(int64_t m, int64_t n) {
    if (m <= 0 || n <= 0 || m % kTile || n % kTile) return fail(QTIP_ERR_SHAPE, "m and n must be positive multiples of 16");
    return QTIP_OK;
}
}  // namespace

// Error / code-argument helpers for the other translation units' extern "C" entry points (k_chain.cu).
qtip_status api_fail(qtip_status s, const char* msg) { return fail(s, msg); }
qtip_status api_cuda_fail(cudaError_t e, const char* where) { return cuda_fail(e, where); }
CodeArgs api_code_args(const qtip_params* p) { return code_args(p); }

void count_launch(int n) { g_launches += (uint64_t)n; }

bool g_pdl = true;
bool g_fused_reduce = false;
bool g_layer_auto = false;     // auto-pick the fused layer kernel (knob 3)
int g_l2_prefetch = 0;         // knob 4: RHT-in L2-prefetches up to this many MiB of the layer's weights (0 = off;
                               // measured: 542 -> 536 GB/s 3INST, 1153 -> 1124 HYB at 64 MiB, profiles/r2s3/)
bool pdl_enabled() { return g_pdl; }

void prefer_max_smem(const void* kern) {
    static std::mutex mu;
    static std::unordered_set<const void*> done;
    std::lock_guard<std::mutex> lock(mu);
    if (done.insert(kern).second)
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
}

int num_sms() {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

}  // namespace qtip

using namespace qtip;

extern "C" {

void qtip_params_default(qtip_params* p, int32_t code, int32_t k) {
    std::memset(p, 0, sizeof(*p));
    p->L = 16;
    p->k = k;
    p->code = code;
    p->V = (code == QTIP_CODE_HYB) ? 2 : 1;
    p->Q = 9;
    p->tail_biting = 1;
    p->Tx = p->Ty = 16;
    if (code == QTIP_CODE_1MAD) { p->lcg_a = 34038481u; p->lcg_b = 76625530u; }
    if (code == QTIP_CODE_3INST) { p->lcg_a = 89226354u; p->lcg_b = 64248484u; }
    p->m_fp16 = 0x3B60u;                                                            // fp16(0.922)
    p->hyb_two_sign = 0;
    if (code == QTIP_CODE_LUT) {
        p->L = 14;
        p->Tx = 32;
        p->Ty = 8;
    }
}

qtip_status qtip_params_check(const qtip_params* p) {
    if (!p) return fail(QTIP_ERR_INVALID_PARAMS, "params is NULL");
    if (p->code != QTIP_CODE_1MAD && p->code != QTIP_CODE_3INST && p->code != QTIP_CODE_HYB && p->code != QTIP_CODE_LUT)
        return fail(QTIP_ERR_INVALID_PARAMS, "unknown code");
    if (p->k < 1 || p->k > 4) return fail(QTIP_ERR_INVALID_PARAMS, "k must be in 1..4");
    if (p->V != 1 && p->V != 2) return fail(QTIP_ERR_INVALID_PARAMS, "V must be 1 or 2");
    if (p->code != QTIP_CODE_HYB && p->V != 1) return fail(QTIP_ERR_INVALID_PARAMS, "1MAD/3INST/LUT need V=1, HYB V=2 (or 1)");
    if (p->L < p->k * p->V || p->L > 32) return fail(QTIP_ERR_INVALID_PARAMS, "need kV <= L <= 32");
    if (p->code == QTIP_CODE_HYB && (p->Q < 1 || p->Q > 15)) return fail(QTIP_ERR_INVALID_PARAMS, "HYB needs 1 <= Q <= 15");
    if (p->Tx * p->Ty != 256 || p->Tx < 1 || p->Ty < 1) return fail(QTIP_ERR_INVALID_PARAMS, "need Tx * Ty = T = 256");
    if (!p->tail_biting) return fail(QTIP_ERR_UNSUPPORTED, "device path needs tail-biting tiles (kT bits)");
    if (p->code == QTIP_CODE_LUT) {
        if (p->L > 16) return fail(QTIP_ERR_UNSUPPORTED, "LUT code: L <= 16 (a 2^L binary16 table in shared memory)");
        if (!((p->Tx == 16 && p->Ty == 16) || (p->Tx == 32 && p->Ty == 8)))
            return fail(QTIP_ERR_UNSUPPORTED, "LUT code: T_x x T_y = 16 x 16 or 32 x 8 (PAPER.md:787)");
        return QTIP_OK;
    }
    if (p->L != 16) return fail(QTIP_ERR_UNSUPPORTED, "device path implements L = 16 (PAPER.md:415, :573)");
    if (p->Tx != 16 || p->Ty != 16) return fail(QTIP_ERR_UNSUPPORTED, "device path needs Tx = Ty = 16 (32 x 8: the LUT code)");
    if (p->code == QTIP_CODE_HYB && p->V == 1 && (p->Q > 14 || p->hyb_two_sign))
        return fail(QTIP_ERR_UNSUPPORTED, "HYB with V = 1: Q <= 14, one sign (PAPER.md:607-609)");
    return QTIP_OK;
}

int64_t qtip_packed_bytes(const qtip_params* p, int64_t m, int64_t n) {
    if (qtip_params_check(p) != QTIP_OK || check_shape(m, n) != QTIP_OK) return -1;
    const Layout l = make_layout(m, n, p->k);
    return l.n_rb * l.n_kc * l.cell_words * 4;
}

qtip_status qtip_pack(const qtip_params* p, int64_t m, int64_t n, const uint8_t* h_tiles, void* d_packed,
                      void* stream) {
    qtip_status st = qtip_params_check(p);
    if (st != QTIP_OK) return st;
    if ((st = check_shape(m, n)) != QTIP_OK) return st;
    if (!h_tiles || !d_packed) return fail(QTIP_ERR_INVALID_PARAMS, "NULL buffer");
    if (!aligned16(d_packed)) return fail(QTIP_ERR_ALIGNMENT, "d_packed must be 16-byte aligned");
    if ((st = check_block(p, m, n)) != QTIP_OK) return st;
    const Layout l = make_layout(m, n, p->k);
    const int64_t tile_bytes = 4 * l.tw;
    // T_x x T_y blocks: block (I_l, J_l) of a cell goes to slot s = I_l (128 / T_y) + J_l, stored at
    // the 16 x 16 position (s / 8, s % 8) (for 16 x 16 blocks: (I_l, J_l) itself)
    const int cr = kCellRows / p->Tx, cc = kCellCols / p->Ty;
    const int64_t mt = m / p->Tx, nt = n / p->Ty;
    std::vector<uint32_t> buf((size_t)(l.n_rb * l.n_kc * l.cell_words), 0u);
    auto work = [&](int64_t t0, int64_t t1) {
        for (int64_t Ig = t0; Ig < t1; ++Ig) {
            const int64_t RB = Ig / cr;
            const int Il = (int)(Ig % cr);
            for (int64_t Jg = 0; Jg < nt; ++Jg) {
                const int64_t KC = Jg / cc;
                const int slot = Il * cc + (int)(Jg % cc);
                const int I = slot >> 3, J = slot & 7;
                const uint8_t* src = h_tiles + (Ig * nt + Jg) * tile_bytes;
                uint32_t* cell = buf.data() + (RB * l.n_kc + KC) * l.cell_words;
                for (int w = 0; w < l.tw; ++w) {
                    const uint8_t* b = src + 4 * w;
                    cell[cell_word_index(I, J, w, l.tw)] =
                        ((uint32_t)b[0] << 24) | ((uint32_t)b[1] << 16) | ((uint32_t)b[2] << 8) | (uint32_t)b[3];
                }
            }
        }
    };
    const int nthreads = (int)std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()), std::max<int64_t>(1, mt / 64));
    if (nthreads <= 1) {
        work(0, mt);
    } else {
        std::vector<std::thread> th;
        for (int i = 0; i < nthreads; ++i) th.emplace_back(work, mt * i / nthreads, mt * (i + 1) / nthreads);
        for (auto& t : th) t.join();
    }
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemcpyAsync(d_packed, buf.data(), buf.size() * 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "qtip_pack copy");
    return QTIP_OK;
}

qtip_status qtip_pack_states(const qtip_params* p, int64_t m, int64_t n, const uint32_t* h_states, void* d_packed,
                             void* stream) {
    qtip_status st = qtip_params_check(p);
    if (st != QTIP_OK) return st;
    if ((st = check_shape(m, n)) != QTIP_OK) return st;
    if (!h_states) return fail(QTIP_ERR_INVALID_PATH, "NULL states");
    const int L = p->L, kv = p->k * p->V, steps = 256 / p->V;
    const uint32_t lmask = (L == 32) ? 0xFFFFFFFFu : ((1u << L) - 1u);
    const uint32_t omask = (1u << (L - kv)) - 1u;
    if ((st = check_block(p, m, n)) != QTIP_OK) return st;
    const int64_t ntiles = (m / p->Tx) * (n / p->Ty);
    const int tile_bytes = p->k * 32;
    std::vector<uint8_t> bytes((size_t)(ntiles * tile_bytes), 0);
    for (int64_t t = 0; t < ntiles; ++t) {
        const uint32_t* s = h_states + t * steps;
        uint8_t* out = bytes.data() + t * tile_bytes;
        for (int q = 0; q < steps; ++q) {
            const uint32_t cur = s[q], nxt = s[(q + 1) % steps];
            if (cur & ~lmask) return fail(QTIP_ERR_INVALID_PATH, "state out of range");
            // edge rule; for q = steps-1 this is the tail-biting closure
            if ((nxt >> kv) != (cur & omask)) return fail(QTIP_ERR_INVALID_PATH, "edge rule / tail-biting closure violated");
            // stream bits [q kV, (q+1) kV) are the top kV bits of state q
            const uint32_t top = cur >> (L - kv);
            for (int i = 0; i < kv; ++i) {
                const int bit = q * kv + i;
                if ((top >> (kv - 1 - i)) & 1u) out[bit >> 3] |= (uint8_t)(0x80u >> (bit & 7));
            }
        }
    }
    return qtip_pack(p, m, n, bytes.data(), d_packed, stream);
}

qtip_status qtip_decode(const qtip_params* p, int64_t m, int64_t n, const void* d_packed, const uint16_t* d_lut,
                        int out_dtype, void* d_out, void* stream) {
    qtip_status st = qtip_params_check(p);
    if (st != QTIP_OK) return st;
    if ((st = check_shape(m, n)) != QTIP_OK) return st;
    if (!d_packed || !d_out || ((p->code == QTIP_CODE_HYB || p->code == QTIP_CODE_LUT) && !d_lut))
        return fail(QTIP_ERR_INVALID_PARAMS, "NULL buffer");
    if (out_dtype != 0 && out_dtype != 1) return fail(QTIP_ERR_INVALID_PARAMS, "out_dtype must be 0 or 1");
    if (!aligned16(d_packed) || !aligned16(d_out)) return fail(QTIP_ERR_ALIGNMENT, "buffers must be 16-byte aligned");
    if ((st = check_block(p, m, n)) != QTIP_OK) return st;
    const Layout l = make_layout(m, n, p->k);
    if (is_variant(p)) {
        const cudaError_t ev = launch_variant_decode(p, l, d_packed, d_lut, out_dtype, d_out, (cudaStream_t)stream);
        if (ev != cudaSuccess) return cuda_fail(ev, "qtip_decode");
        return QTIP_OK;
    }
    cudaError_t e = launch_decode(l, p->code, p->V, code_args(p), d_packed, d_lut, out_dtype, d_out, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "qtip_decode");
    return QTIP_OK;
}

static size_t align256(size_t x) { return (x + 255) / 256 * 256; }

// Workspace regions (one caller buffer per layer, 256-B aligned).
struct WsLayout {
    size_t xt, partial, yt, cnt, lws, bar, seg, total;
};
static WsLayout ws_layout(const qtip_params* p, const Layout& l, int64_t B) {
    WsLayout o;
    const int64_t Bx = B <= 8 ? 8 : (B <= 16 ? 16 : 64);          // x~ rows (batch pad of the kernels)
    size_t off = 0;
    o.xt = off;
    off += align256(4 * Bx * l.n_pad);
    o.partial = off;
    off += align256(4 * l.n_kc * B * l.m_pad);
    o.yt = off;
    off += align256(4 * B * l.m_pad);
    o.cnt = off;
    off += align256(4 * (l.m_pad / kCellRows + 2));
    o.lws = off;
    off += align256(4 * layer_workspace_floats(l, B, 0));
    o.bar = off;
    off += 1024;
    o.seg = off;
    off += align256(4 * umma_seg_floats(l, p->code, B));
    o.total = off;
    return o;
}

// Profile events also work inside CUDA-graph capture (as external event-record nodes).
static void record_event(cudaEvent_t ev, cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive)
        cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal);
    else
        cudaEventRecord(ev, s);
}

// The auto kernel choice depends on (p, m, n, B) and the group size only -- never on the row range
// of a call -- so QTIP_XT_READY reuses an x~ written in the same layout.
static bool use_umma(const qtip_params* p, const Layout& l, int64_t B, int G) {
    if (g_impl != 0 && g_impl != 7) return false;
    if (!umma_supported(l, p->code, code_args(p), B, G)) return false;
    if (g_impl == 7) return true;
    // auto (measured, profiles/r2_*): the tcgen05 stream-K kernel wins for HYB at batch
    // 1-8 once every SM has >= 10 cells of the launch (q,k,v / gate,up groups and the 11008-wide
    // layers); short single launches keep the row-tile kernel (fixed start-up + stream-K fix-up cost).
    // For 3INST / 1MAD the decode (5 instructions per weight), not the MMA, bounds it: only the 70B
    // layers (>= 40 cells per SM) gain (C4 8192 x 28672: 69.6 -> 66.7 us)
    // 3INST / 1MAD at batch >= 8: impl 7 beats the split-K / CUDA-core kernels on the 7B step at every
    // measured batch (B = 8 / 16 / 32: 265 -> 300, 160 -> 193, 42 -> 70 GB/s, profiles/r2/batch_*)
    // HYB at any batch once every SM has >= 10 cells: the x~ slab ring (round 2) removed the batch
    // limit (B = 16: q,k,v 39.1 -> 27.4 us, gate,up 62.1 -> 28.9 us, down 33.0 -> 23.0 us vs the
    // split-K kernel, profiles/r2s3/)
    const int64_t cells = (int64_t)G * l.n_rb * l.n_kc;
    if (p->code != QTIP_CODE_HYB && B >= 8) return true;
    // 3INST at batch 1-7: >= 20 cells per SM (the grouped q,k,v and gate,up launches: 17.6 -> 17.2 us,
    // 26.8 -> 25.6 us with the selector pair sum; single 4096-row layers keep impls 3/4); 1MAD >= 40
    // (its 7B step lost 534 -> 521 GB/s at 20)
    const int64_t min_cells = (p->code == QTIP_CODE_HYB ? 10 : p->code == QTIP_CODE_3INST ? 20 : 40) * (int64_t)num_sms();
    return (p->code == QTIP_CODE_HYB || B <= 8) && cells >= min_cells;
}

// The RHT-in launch that precedes a GEMV prefetches the GEMV's weights (row blocks [rb0, rb1) of
// each layer, at most g_l2_prefetch MiB per layer) into L2 before its PDL wait (DESIGN 5.4).
static void prefetch_weights(const Layout& l, int G, const void* const* packed, int64_t rb0, int64_t rb1) {
    if (g_l2_prefetch <= 0) return;
    const void* ptr[kMaxGroup];
    uint64_t bytes[kMaxGroup];
    const uint64_t cellb = (uint64_t)l.cell_words * 4u, cap = (uint64_t)g_l2_prefetch << 20;
    for (int g = 0; g < G; ++g) {
        ptr[g] = (const char*)packed[g] + (uint64_t)rb0 * (uint64_t)l.n_kc * cellb;
        const uint64_t b = (uint64_t)(rb1 - rb0) * (uint64_t)l.n_kc * cellb;
        bytes[g] = b < cap ? b : cap;
    }
    rht_set_prefetch(G, ptr, bytes);
}

int qtip_matvec_group_fused(const qtip_params* p, int G, int64_t m, int64_t n, int64_t B) {
    if (G < 2 || G > kMaxGroup || qtip_params_check(p) != QTIP_OK || check_shape(m, n) != QTIP_OK || B < 1 || B > 64)
        return 0;
    if (is_variant(p)) return 0;                                   // per-layer calls (k_variant.cu)
    const Layout l = make_layout(m, n, p->k);
    if (use_umma(p, l, B, G)) return 1;
    if (!(g_impl == 0 || g_impl == 6)) return 0;
    // measured: HYB at B >= 4 runs faster as concurrent per-layer row-tile kernels
    if (g_impl == 0 && p->code == QTIP_CODE_HYB && B >= 4) return 0;
    return layer_group_supported(l, p->code, code_args(p), B, G) ? 1 : 0;
}

qtip_status qtip_matvec_group(const qtip_params* p, int G, int64_t m, int64_t n, int64_t B,
                              const void* const* d_packed, const uint16_t* const* d_lut, const uint8_t* const* d_sign_n,
                              const uint8_t* const* d_sign_m, const float* scale, const float* d_x, float* const* d_y,
                              int flags, void* const* d_workspace, size_t workspace_bytes, void* stream) {
    if (G < 1 || G > kMaxGroup) return fail(QTIP_ERR_INVALID_PARAMS, "group size must be in 1..4");
    if (!d_packed || !d_y || !d_workspace || !scale || !d_sign_n || !d_sign_m)
        return fail(QTIP_ERR_INVALID_PARAMS, "NULL pointer array");
    // every member's arguments are validated by the per-layer entry point's rules
    qtip_status st = qtip_params_check(p);
    if (st != QTIP_OK) return st;
    if ((st = check_shape(m, n)) != QTIP_OK) return st;
    if (B < 1 || B > 64) return fail(QTIP_ERR_INVALID_PARAMS, "batch must be in 1..64");
    if (flags & ~(QTIP_RHT_IN | QTIP_RHT_OUT | QTIP_XT_READY)) return fail(QTIP_ERR_INVALID_PARAMS, "unknown flags");
    const size_t need = qtip_matvec_workspace_bytes(p, m, n, B);
    for (int g = 0; g < G; ++g) {
        if (!d_packed[g] || !d_y[g] || !d_workspace[g] || !d_x || (p->code == QTIP_CODE_HYB && (!d_lut || !d_lut[g])))
            return fail(QTIP_ERR_INVALID_PARAMS, "NULL buffer");
        if (((flags & QTIP_RHT_IN) && !(flags & QTIP_XT_READY) && !d_sign_n[g]) || ((flags & QTIP_RHT_OUT) && !d_sign_m[g]))
            return fail(QTIP_ERR_INVALID_PARAMS, "NULL sign vector");
        if (!aligned16(d_packed[g]) || (reinterpret_cast<uintptr_t>(d_workspace[g]) & 255u))
            return fail(QTIP_ERR_ALIGNMENT, "d_packed 16-B and d_workspace 256-B aligned");
        if (workspace_bytes < need) return fail(QTIP_ERR_WORKSPACE, "workspace too small");
    }
    const Layout l = make_layout(m, n, p->k);
    const CodeArgs ca = code_args(p);
    const bool rin = (flags & QTIP_RHT_IN) != 0, rout = (flags & QTIP_RHT_OUT) != 0;
    const bool xready = (flags & QTIP_XT_READY) != 0;
    bool grouped = qtip_matvec_group_fused(p, G, m, n, B) != 0;
    const bool umma = grouped && use_umma(p, l, B, G);
    if (umma && p->code == QTIP_CODE_HYB)                        // one shared-memory LUT per launch
        for (int g = 1; g < G; ++g)
            if (d_lut[g] != d_lut[0]) grouped = false;
    if (!grouped) {                                              // one layer at a time (same results)
        for (int g = 0; g < G; ++g) {
            st = qtip_matvec(p, m, n, B, d_packed[g], d_lut ? d_lut[g] : nullptr, d_sign_n[g], d_sign_m[g], scale[g], d_x, d_y[g], 0, m,
                             flags, d_workspace[g], workspace_bytes, stream);
            if (st != QTIP_OK) return st;
        }
        return QTIP_OK;
    }
    RhtPlan pn{}, pm{};
    if (rin && !xready && make_rht_plan(n, &pn, 128 / G, B) != cudaSuccess) return fail(QTIP_ERR_SHAPE, "no supported Hadamard order for n");
    if (rout && make_rht_plan(m, &pm, 128 / G, B) != cudaSuccess) return fail(QTIP_ERR_SHAPE, "no supported Hadamard order for m");
    cudaStream_t s = (cudaStream_t)stream;
    const WsLayout o = ws_layout(p, l, B);
    const float* xin[kMaxGroup];
    void* xt[kMaxGroup];
    for (int g = 0; g < G; ++g) {
        xt[g] = (char*)d_workspace[g] + o.xt;
        xin[g] = d_x;
    }
    cudaError_t e = cudaSuccess;
    if (umma) {
        // grouped RHT-in -> one stream-K tcgen05 launch over the G layers' cells -> grouped RHT-out
        // (or segment reduction) reading the partial-sum segments
        const int xmode = umma_xt_mode(p->code);
        const int64_t bp = umma_batch_pad(B);
        int* tk0[kMaxGroup];                                       // the GEMV's row-block tickets: cleared here
        for (int g = 0; g < G; ++g) tk0[g] = (int*)((char*)d_workspace[g] + o.cnt);
        if (!xready) {
            if (rin) {
                prefetch_weights(l, G, d_packed, 0, l.n_rb);
                e = launch_rht_group(pn, G, B, d_sign_n, xin, n, xt, bp, 0, std::vector<float>(G, 1.0f).data(), s, xmode,
                                     l.n_pad, tk0, (int)l.n_rb);
            } else {
                for (int g = 0; g < G && e == cudaSuccess; ++g)
                    e = launch_convert(d_x, n, n, B, xt[g], bp, xmode, l.n_pad, s, tk0[g], (int)l.n_rb);
            }
            if (e != cudaSuccess) return cuda_fail(e, "qtip_matvec_group rht_in");
        }
        float* segs[kMaxGroup];
        int* tks[kMaxGroup];
        float* yo[kMaxGroup];
        float ysc[kMaxGroup];
        for (int g = 0; g < G; ++g) {
            segs[g] = (float*)((char*)d_workspace[g] + o.seg);
            tks[g] = (int*)((char*)d_workspace[g] + o.cnt);
            yo[g] = rout ? (float*)((char*)d_workspace[g] + o.yt) : d_y[g];
            ysc[g] = rout ? 1.0f : scale[g];
        }
        const bool prof = g_prof_start && g_prof_stop;
        if (prof) record_event(g_prof_start, s);
        e = launch_umma(l, p->code, ca, G, d_packed, d_lut ? d_lut[0] : nullptr, (const void* const*)xt, segs, tks, yo, ysc,
                        rout ? l.m_pad : m, m, B, 0, l.n_rb, s);
        if (prof) {
            record_event(g_prof_stop, s);
            g_prof_start = g_prof_stop = nullptr;
        }
        if (e != cudaSuccess) return cuda_fail(e, "qtip_matvec_group gemv");
        if (rout) {
            const float* yin[kMaxGroup];
            void* yout[kMaxGroup];
            for (int g = 0; g < G; ++g) {
                yin[g] = yo[g];
                yout[g] = d_y[g];
            }
            e = launch_rht_group(pm, G, B, d_sign_m, yin, l.m_pad, yout, m, 1, scale, s);
            if (e != cudaSuccess) return cuda_fail(e, "qtip_matvec_group rht_out");
        }
        return QTIP_OK;
    }
    const int64_t Bx = B <= 8 ? 8 : (B <= 16 ? 16 : B);
    (void)Bx;
    const int xmode = gemv_mma_xt_mode(p->code);
    const int xmode6 = p->code == QTIP_CODE_HYB ? 5 : xmode;        // HYB fast path: swapped pairs
    const int64_t row_words = l.n_pad * ((xmode == 1 || xmode == 3) ? 4 : 2) / 4;
    float* yt[kMaxGroup];
    float* lws[kMaxGroup];
    unsigned* bar[kMaxGroup];
    float* ydst[kMaxGroup];
    float sc[kMaxGroup];
    for (int g = 0; g < G; ++g) {                                 // the impl 6 workspace layout
        char* ws = (char*)d_workspace[g];
        yt[g] = (float*)(ws + o.yt);
        lws[g] = (float*)(ws + o.lws);
        bar[g] = (unsigned*)(ws + o.bar);
        ydst[g] = rout ? yt[g] : d_y[g];
        sc[g] = rout ? 1.0f : scale[g];
    }
    if (!xready) {                                                // also clears the barrier / ticket words
        if (rin) {
            prefetch_weights(l, G, d_packed, 0, l.n_rb);
            e = launch_rht_group(pn, G, B, d_sign_n, xin, n, xt, l.n_pad, 0, std::vector<float>(G, 1.0f).data(), s,
                                 xmode6, l.n_pad, (int* const*)bar, 256);
        } else {
            for (int g = 0; g < G && e == cudaSuccess; ++g)
                e = launch_convert(d_x, n, n, B, xt[g], l.n_pad, xmode6, l.n_pad, s, (int*)bar[g], 256);
        }
        if (e != cudaSuccess) return cuda_fail(e, "qtip_matvec_group rht_in");
    }
    const uint16_t* luts[kMaxGroup];
    for (int g = 0; g < G; ++g) luts[g] = d_lut ? d_lut[g] : nullptr;
    e = launch_layer_group(l, p->code, ca, G, d_packed, luts, sc, ydst, B, (uint32_t* const*)xt, row_words, lws, bar, s);
    if (e != cudaSuccess) return cuda_fail(e, "qtip_matvec_group gemv");
    if (rout) {
        const float* yin[kMaxGroup];
        void* yout[kMaxGroup];
        for (int g = 0; g < G; ++g) {
            yin[g] = yt[g];
            yout[g] = d_y[g];
        }
        e = launch_rht_group(pm, G, B, d_sign_m, yin, m, yout, m, 1, scale, s);
        if (e != cudaSuccess) return cuda_fail(e, "qtip_matvec_group rht_out");
    }
    return QTIP_OK;
}

size_t qtip_matvec_workspace_bytes(const qtip_params* p, int64_t m, int64_t n, int64_t B) {
    if (qtip_params_check(p) != QTIP_OK || check_shape(m, n) != QTIP_OK || B < 1) return 0;
    return ws_layout(p, make_layout(m, n, p->k), B).total;
}

qtip_status qtip_matvec(const qtip_params* p, int64_t m, int64_t n, int64_t B, const void* d_packed,
                        const uint16_t* d_lut, const uint8_t* d_sign_n, const uint8_t* d_sign_m, float scale,
                        const float* d_x, float* d_y, int64_t row_begin, int64_t row_end, int flags,
                        void* d_workspace, size_t workspace_bytes, void* stream) {
    qtip_status st = qtip_params_check(p);
    if (st != QTIP_OK) return st;
    if ((st = check_shape(m, n)) != QTIP_OK) return st;
    if (B < 1 || B > 64) return fail(QTIP_ERR_INVALID_PARAMS, "batch must be in 1..64");
    if (flags & ~(QTIP_RHT_IN | QTIP_RHT_OUT | QTIP_XT_READY)) return fail(QTIP_ERR_INVALID_PARAMS, "unknown flags");
    if (!d_packed || !d_x || !d_y || !d_workspace || ((p->code == QTIP_CODE_HYB || p->code == QTIP_CODE_LUT) && !d_lut))
        return fail(QTIP_ERR_INVALID_PARAMS, "NULL buffer");
    if (((flags & QTIP_RHT_IN) && !(flags & QTIP_XT_READY) && !d_sign_n) || ((flags & QTIP_RHT_OUT) && !d_sign_m))
        return fail(QTIP_ERR_INVALID_PARAMS, "NULL sign vector");
    if (row_begin < 0 || row_end > m || row_begin >= row_end) return fail(QTIP_ERR_SHAPE, "bad row range");
    if (row_begin % kCellRows || (row_end % kCellRows && row_end != m))
        return fail(QTIP_ERR_SHAPE, "row_begin/row_end must be multiples of 128 (or row_end == m)");
    if ((row_begin != 0 || row_end != m) && (flags & QTIP_RHT_OUT))
        return fail(QTIP_ERR_INVALID_PARAMS, "a partial row range needs QTIP_RHT_OUT off (H_m^T mixes all rows)");
    if (!aligned16(d_packed) || (reinterpret_cast<uintptr_t>(d_workspace) & 255u))
        return fail(QTIP_ERR_ALIGNMENT, "d_packed 16-B and d_workspace 256-B aligned");
    const size_t need = qtip_matvec_workspace_bytes(p, m, n, B);
    if (workspace_bytes < need) return fail(QTIP_ERR_WORKSPACE, "workspace too small");
    RhtPlan pn{}, pm{};
    if ((flags & QTIP_RHT_IN) && !(flags & QTIP_XT_READY) && make_rht_plan(n, &pn, 128, B) != cudaSuccess)
        return fail(QTIP_ERR_SHAPE, "no supported Hadamard order for n");
    if ((flags & QTIP_RHT_OUT) && make_rht_plan(m, &pm, 128, B) != cudaSuccess)
        return fail(QTIP_ERR_SHAPE, "no supported Hadamard order for m");

    const Layout l = make_layout(m, n, p->k);
    const CodeArgs ca = code_args(p);
    cudaStream_t s = (cudaStream_t)stream;
    const WsLayout o = ws_layout(p, l, B);
    char* ws = (char*)d_workspace;
    void* xt = ws + o.xt;
    const bool rin = (flags & QTIP_RHT_IN) != 0, rout = (flags & QTIP_RHT_OUT) != 0;
    const int64_t rb0 = row_begin / kCellRows, rb1 = (row_end + kCellRows - 1) / kCellRows;
    cudaError_t e;
    if (is_variant(p)) {
        // the NEXT-3 code variants (k_variant.cu): RHT-in -> fused decode-GEMV with the whole table
        // in shared memory -> fixed-order split-K reduction -> RHT-out
        if ((st = check_block(p, m, n)) != QTIP_OK) return st;
        if (variant_gemv_smem(p, B) > 227 * 1024) return fail(QTIP_ERR_UNSUPPORTED, "table + x~ slice exceed shared memory");
        float* vpart = (float*)(ws + o.partial);
        float* vyt = (float*)(ws + o.yt);
        e = cudaSuccess;
        if (!(flags & QTIP_XT_READY)) {
            if (rin) e = launch_rht(pn, B, d_sign_n, d_x, n, xt, l.n_pad, 0, 1.0f, s, 0, l.n_pad);
            else e = launch_convert(d_x, n, n, B, xt, l.n_pad, 0, l.n_pad, s);
        }
        if (e != cudaSuccess) return cuda_fail(e, "qtip_matvec rht_in");
        const bool prof = g_prof_start && g_prof_stop;
        if (prof) record_event(g_prof_start, s);
        e = launch_variant_gemv(p, l, d_packed, d_lut, (const float*)xt, B, rb0, rb1, vpart, s);
        if (prof) {
            record_event(g_prof_stop, s);
            g_prof_start = g_prof_stop = nullptr;
        }
        if (e != cudaSuccess) return cuda_fail(e, "qtip_matvec variant gemv");
        if (rout) {
            e = launch_reduce(vpart, l.n_kc, B, l.m_pad, 0, m, 1.0f, vyt, l.m_pad, s);
            if (e == cudaSuccess) e = launch_rht(pm, B, d_sign_m, vyt, l.m_pad, d_y, m, 1, scale, s);
        } else {
            e = launch_reduce(vpart, l.n_kc, B, l.m_pad, row_begin, row_end, scale, d_y, row_end - row_begin, s);
        }
        if (e != cudaSuccess) return cuda_fail(e, "qtip_matvec epilogue");
        return QTIP_OK;
    }
    const bool umma_ok = umma_supported(l, p->code, ca, B, 1);
    if (g_impl == 7 && !umma_ok)
        return fail(QTIP_ERR_UNSUPPORTED, "tcgen05 stream-K kernel: needs 2 <= k <= 4, B <= 64, HYB Q = 9 one-sign");
    if (use_umma(p, l, B, 1)) {
        // impl 7 (auto default): RHT-in -> stream-K tcgen05 decode-GEMV (k_umma.cu) -> RHT-out reading
        // the partial-sum segments (or the segment reduction when RHT-out is off)
        const int xmode = umma_xt_mode(p->code);
        const int64_t bp = umma_batch_pad(B);
        e = cudaSuccess;
        int* tk0 = (int*)(ws + o.cnt);                   // the GEMV's row-block tickets: cleared here
        const int ntk = (int)(rb1 - rb0);
        if (!(flags & QTIP_XT_READY)) {
            if (rin) {
                prefetch_weights(l, 1, &d_packed, rb0, rb1);
                e = launch_rht(pn, B, d_sign_n, d_x, n, xt, bp, 0, 1.0f, s, xmode, l.n_pad, tk0, ntk);
            }
            else e = launch_convert(d_x, n, n, B, xt, bp, xmode, l.n_pad, s, tk0, ntk);
        }
        if (e != cudaSuccess) return cuda_fail(e, "qtip_matvec rht_in");
        float* segp = (float*)(ws + o.seg);
        int* tk = (int*)(ws + o.cnt);
        float* yo = rout ? (float*)(ws + o.yt) : d_y;
        const float ysc = rout ? 1.0f : scale;
        const int64_t rows = row_end - row_begin;
        const bool prof = g_prof_start && g_prof_stop;
        if (prof) record_event(g_prof_start, s);
        e = launch_umma(l, p->code, ca, 1, &d_packed, d_lut, (const void* const*)&xt, &segp, &tk, &yo, &ysc,
                        rout ? l.m_pad : rows, rows, B, rb0, rb1, s);
        if (prof) {
            record_event(g_prof_stop, s);
            g_prof_start = g_prof_stop = nullptr;
        }
        if (e != cudaSuccess) return cuda_fail(e, "qtip_matvec gemv");
        if (rout) e = launch_rht(pm, B, d_sign_m, yo, l.m_pad, d_y, m, 1, scale, s);
        if (e != cudaSuccess) return cuda_fail(e, "qtip_matvec rht_out");
        return QTIP_OK;
    }
    // kernel choice: 1 CUDA-core reference, 2 tcgen05 (A in TMEM), 3 register-fed mma.sync;
    // auto picks the measured-fastest supported one
    const bool tc_ok = gemv_tc_supported(l, p->code, ca, B);
    const bool mma_ok = gemv_mma_supported(l, p->code, ca, B);
    const bool row_ok = gemv_row_supported(l, p->code, ca, B);
    if (g_impl == 2 && !tc_ok) return fail(QTIP_ERR_UNSUPPORTED, "tcgen05 kernel: needs 2 <= k <= 4, B <= 16, HYB Q = 9 one-sign");
    if (g_impl == 3 && !mma_ok) return fail(QTIP_ERR_UNSUPPORTED, "mma kernel: needs 2 <= k <= 4, B <= 16, one-sign HYB");
    if (g_impl == 4 && !row_ok) return fail(QTIP_ERR_UNSUPPORTED, "row kernel: needs 2 <= k <= 4, B <= 4, one-sign HYB");
    const int64_t launch_tile_rows = (row_end - row_begin + kTile - 1) / kTile;
    const bool layer_ok = layer_supported(l, p->code, ca, B, launch_tile_rows, rin && !(flags & QTIP_XT_READY), rout);
    if (g_impl == 5 && !layer_ok)
        return fail(QTIP_ERR_UNSUPPORTED, "fused layer kernel: needs 2 <= k <= 4, B <= 4, one-sign HYB, shared memory fit");
    const bool gemv6_ok = layer_supported(l, p->code, ca, B, launch_tile_rows, false, false);
    if (g_impl == 6 && !gemv6_ok)
        return fail(QTIP_ERR_UNSUPPORTED, "persistent GEMV kernel: needs 2 <= k <= 4, B <= 4, one-sign HYB, shared memory fit");
    int impl = g_impl;
    if (impl == 0 && layer_ok && g_layer_auto) impl = 5;
    // Fallback when impl 7 does not apply (two-sign HYB, Q != 9, B > 64 is refused anyway): the
    // choice uses the FULL layer's tile rows, so a row shard takes the same kernel (and the same
    // x~ layout for QTIP_XT_READY) as the full call.
    // measured: for HYB at batch 1 the persistent GEMV with the shared-memory
    // LUT fast path (impl 6) beats the row-tile and split-K kernels (at B = 4 it does not)
    const bool one_wave = l.m / kTile <= 2 * (int64_t)num_sms();
    const bool gemv6_full = layer_supported(l, p->code, ca, B, l.m / kTile, false, false);
    if (impl == 0 && gemv6_full && gemv6_ok && p->code == QTIP_CODE_HYB && B == 1 && !(one_wave && n <= 8192)) impl = 6;
    if (impl == 0) impl = (row_ok && one_wave) ? 4 : (mma_ok ? 3 : (tc_ok ? 2 : 1));
    const bool use_tc = impl == 2, use_mma = impl == 3, use_row = impl == 4;
    float* partial = (float*)(ws + o.partial);
    float* yt = (float*)(ws + o.yt);
    int* cnt = (int*)(ws + o.cnt);
    const int n_rb = (int)(l.m_pad / kCellRows);
    const int xmode = (use_mma || use_row || impl == 5 || impl == 6) ? gemv_mma_xt_mode(p->code) : (use_tc ? gemv_tc_xt_mode(p->code) : 0);
    float* lws = (float*)(ws + o.lws);
    unsigned* bar = (unsigned*)(ws + o.bar);
    if (impl == 6) {
        // RHT-in kernel -> persistent row-owning decode-GEMV (k_layer.cu without its RHT phases,
        // x~ from the workspace) -> RHT-out kernel
        const int64_t row_words = l.n_pad * ((xmode == 1 || xmode == 3) ? 4 : 2) / 4;
        const int xmode6 = p->code == QTIP_CODE_HYB ? 5 : xmode;   // HYB fast path: swapped pairs
        e = cudaSuccess;
        if (!(flags & QTIP_XT_READY)) {                          // also clears the barrier / ticket words
            if (rin) {
                prefetch_weights(l, 1, &d_packed, rb0, rb1);
                e = launch_rht(pn, B, d_sign_n, d_x, n, xt, l.n_pad, 0, 1.0f, s, xmode6, l.n_pad, (int*)bar, 256);
            }
            else e = launch_convert(d_x, n, n, B, xt, l.n_pad, xmode6, l.n_pad, s, (int*)bar, 256);
        }
        if (e != cudaSuccess) return cuda_fail(e, "qtip_matvec rht_in");
        const bool prof = g_prof_start && g_prof_stop;
        if (prof) record_event(g_prof_start, s);
        e = launch_layer(l, p->code, ca, d_packed, d_lut, d_x, d_sign_n, d_sign_m, rout ? 1.0f : scale, rout ? yt : d_y,
                         B, row_begin, row_end, false, false, true, (uint32_t*)xt, row_words, lws, bar, s);
        if (prof) {
            record_event(g_prof_stop, s);
            g_prof_start = g_prof_stop = nullptr;
        }
        if (e != cudaSuccess) return cuda_fail(e, "qtip_matvec gemv");
        if (rout) e = launch_rht(pm, B, d_sign_m, yt, m, d_y, m, 1, scale, s);
        if (e != cudaSuccess) return cuda_fail(e, "qtip_matvec rht_out");
        return QTIP_OK;
    }
    if (impl == 5) {
        // one persistent launch: RHT-in, decode-GEMV, reduction, RHT-out (k_layer.cu); its grid-barrier
        // and ticket words start from zero whatever the caller's workspace held
        if ((e = cudaMemsetAsync(bar, 0, 1024, s)) != cudaSuccess) return cuda_fail(e, "qtip_matvec barrier words");
        const int64_t row_words = l.n_pad * ((xmode == 1 || xmode == 3) ? 4 : 2) / 4;
        const bool prof = g_prof_start && g_prof_stop;
        if (prof) record_event(g_prof_start, s);
        e = launch_layer(l, p->code, ca, d_packed, d_lut, d_x, d_sign_n, d_sign_m, scale, d_y, B, row_begin, row_end,
                         rin, rout, (flags & QTIP_XT_READY) != 0, (uint32_t*)xt, row_words, lws, bar, s);
        if (prof) {
            record_event(g_prof_stop, s);
            g_prof_start = g_prof_stop = nullptr;
        }
        if (e != cudaSuccess) return cuda_fail(e, "qtip_matvec layer");
        return QTIP_OK;
    }
    // the input kernel also clears the GEMV's split-K arrival counters (workspace is caller memory)
    if (flags & QTIP_XT_READY) e = cudaSuccess;          // counters are left zero by every GEMV
    else if (flags & QTIP_RHT_IN) {
        prefetch_weights(l, 1, &d_packed, rb0, rb1);
        e = launch_rht(pn, B, d_sign_n, d_x, n, xt, l.n_pad, 0, 1.0f, s, xmode, l.n_pad, cnt, n_rb + 2);
    }
    else e = launch_convert(d_x, n, n, B, xt, l.n_pad, xmode, l.n_pad, s, cnt, n_rb + 2);
    if (e != cudaSuccess) return cuda_fail(e, "qtip_matvec rht_in");
    const bool prof = g_prof_start && g_prof_stop;
    if (prof) record_event(g_prof_start, s);
    const bool rht_out = (flags & QTIP_RHT_OUT) != 0;
    const bool fused_reduce = use_row || (use_mma && g_fused_reduce);
    if (use_row) {
        const int64_t row_words = l.n_pad * ((xmode == 1 || xmode == 3) ? 4 : 2) / 4;
        e = launch_gemv_row(l, p->code, ca, d_packed, d_lut, xt, row_words, B, row_begin, row_end,
                            rht_out ? yt : d_y, rht_out ? l.m_pad : row_end - row_begin, rht_out ? 0 : row_begin,
                            rht_out ? m : row_end, rht_out ? 1.0f : scale, s);
    } else if (use_mma) {
        // split-K reduction fused into the GEMV: straight to y (no RHT-out) or to y~
        MmaEpilogue ep;
        ep.cnt = cnt;
        ep.n_rb = n_rb;
        ep.y = rht_out ? yt : d_y;
        ep.y_stride = rht_out ? l.m_pad : row_end - row_begin;
        ep.row_lo = rht_out ? 0 : row_begin;
        ep.row_hi = rht_out ? m : row_end;
        ep.scale = rht_out ? 1.0f : scale;
        if (!fused_reduce) ep.y = nullptr;
        const int64_t row_words = l.n_pad * ((xmode == 1 || xmode == 3) ? 4 : 2) / 4;
        e = launch_gemv_mma(l, p->code, ca, d_packed, d_lut, xt, row_words, B, rb0, rb1, partial, ep, s);
    } else if (use_tc) {
        const int64_t row_bytes = l.n_pad * ((xmode == 1 || xmode == 3) ? 4 : 2);
        e = launch_gemv_tc(l, p->code, ca, d_packed, d_lut, xt, row_bytes, B, rb0, rb1, partial, s);
    } else {
        e = launch_gemv_simple(l, p->code, ca, d_packed, d_lut, (const float*)xt, B, rb0, rb1, partial, s);
    }
    if (prof) {
        record_event(g_prof_stop, s);
        g_prof_start = g_prof_stop = nullptr;
    }
    if (e != cudaSuccess) return cuda_fail(e, "qtip_matvec gemv");
    if (rht_out) {
        if (!fused_reduce) e = launch_reduce(partial, l.n_kc, B, l.m_pad, 0, m, 1.0f, yt, l.m_pad, s);
        if (e == cudaSuccess) e = launch_rht(pm, B, d_sign_m, yt, l.m_pad, d_y, m, 1, scale, s);
    } else if (!fused_reduce) {
        e = launch_reduce(partial, l.n_kc, B, l.m_pad, row_begin, row_end, scale, d_y, row_end - row_begin, s);
    }
    if (e != cudaSuccess) return cuda_fail(e, "qtip_matvec epilogue");
    return QTIP_OK;
}

qtip_status qtip_rht(int64_t n, int64_t B, const uint8_t* d_sign, const float* d_in, float* d_out, int inverse,
                     void* stream) {
    if (n <= 0 || B < 1) return fail(QTIP_ERR_SHAPE, "n and B must be positive");
    if (!d_sign || !d_in || !d_out) return fail(QTIP_ERR_INVALID_PARAMS, "NULL buffer");
    if (d_in == d_out) return fail(QTIP_ERR_INVALID_PARAMS, "qtip_rht is out-of-place (d_in != d_out)");
    RhtPlan plan{};
    if (make_rht_plan(n, &plan, 128, B) != cudaSuccess) return fail(QTIP_ERR_SHAPE, "no supported Hadamard order for n");
    cudaError_t e = launch_rht(plan, B, d_sign, d_in, n, d_out, n, inverse ? 1 : 0, 1.0f, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "qtip_rht");
    return QTIP_OK;
}

size_t qtip_viterbi_workspace_bytes(const qtip_params* p, int64_t T) {
    if (qtip_params_check(p) != QTIP_OK || T < 1) return 0;
    return viterbi_workspace_bytes((int)T);
}

qtip_status qtip_viterbi_tailbite(const qtip_params* p, int64_t nseq, int64_t T, const float* d_source,
                                  const uint16_t* d_lut, uint32_t* d_states, float* d_cost, void* d_workspace,
                                  size_t workspace_bytes, void* stream) {
    qtip_status st = qtip_params_check(p);
    if (st != QTIP_OK) return st;
    if (!viterbi_supported(p->code, p->k, p->V, p->L, p->Q, p->hyb_two_sign))
        return fail(QTIP_ERR_UNSUPPORTED,
                    "GPU quantizer: L = 16; 3INST/1MAD V = 1, k in {2, 3, 4}; HYB V = 2, k in {2, 3, 4}, Q = 9, one sign");
    if (nseq < 1 || T < 2 || T > 4096 || nseq > (1 << 30) || T % p->V) return fail(QTIP_ERR_SHAPE, "need nseq >= 1, 2 <= T <= 4096, V | T");
    if (!d_source || !d_states || !d_cost || !d_workspace || (p->code == QTIP_CODE_HYB && !d_lut))
        return fail(QTIP_ERR_INVALID_PARAMS, "NULL buffer");
    if (workspace_bytes < viterbi_workspace_bytes((int)T)) return fail(QTIP_ERR_WORKSPACE, "workspace too small");
    const cudaError_t e = launch_viterbi(p->code, p->k * p->V, code_args(p), d_source, d_lut, (int)nseq, (int)T, d_states,
                                         d_cost, d_workspace, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "qtip_viterbi_tailbite");
    return QTIP_OK;
}

size_t qtip_quantize_workspace_bytes(const qtip_params* p, int64_t m, int64_t n) {
    if (qtip_params_check(p) != QTIP_OK || check_shape(m, n) != QTIP_OK) return 0;
    return align256(viterbi_workspace_bytes(p->Tx * p->Ty)) + align256((size_t)m * n * 4);
}

qtip_status qtip_quantize_matrix(const qtip_params* p, int64_t m, int64_t n, const float* d_W, float source_scale,
                                 const uint16_t* d_lut, uint32_t* d_states, float* d_cost, void* d_workspace,
                                 size_t workspace_bytes, void* stream) {
    qtip_status st = qtip_params_check(p);
    if (st != QTIP_OK) return st;
    if ((st = check_shape(m, n)) != QTIP_OK) return st;
    if ((st = check_block(p, m, n)) != QTIP_OK) return st;
    if (!viterbi_supported(p->code, p->k, p->V, p->L, p->Q, p->hyb_two_sign))
        return fail(QTIP_ERR_UNSUPPORTED,
                    "GPU quantizer: L = 16; 3INST/1MAD V = 1, k in {2, 3, 4}; HYB V = 2, k in {2, 3, 4}, Q = 9, one sign");
    if (!d_W || !d_states || !d_cost || !d_workspace || (p->code == QTIP_CODE_HYB && !d_lut))
        return fail(QTIP_ERR_INVALID_PARAMS, "NULL buffer");
    if (workspace_bytes < qtip_quantize_workspace_bytes(p, m, n)) return fail(QTIP_ERR_WORKSPACE, "workspace too small");
    const int T = p->Tx * p->Ty;
    const int64_t nseq = (m / p->Tx) * (n / p->Ty);
    cudaStream_t s = (cudaStream_t)stream;
    float* seqs = (float*)((char*)d_workspace + align256(viterbi_workspace_bytes(T)));
    cudaError_t e = launch_gather_sequences(d_W, m, n, p->Tx, p->Ty, source_scale, seqs, s);
    if (e == cudaSuccess)
        e = launch_viterbi(p->code, p->k * p->V, code_args(p), seqs, d_lut, (int)nseq, T, d_states, d_cost, d_workspace, s);
    if (e != cudaSuccess) return cuda_fail(e, "qtip_quantize_matrix");
    return QTIP_OK;
}

qtip_status qtip_hadamard_order(int64_t n, int32_t* b, int32_t* a) {
    int bb, aa;
    if (!b || !a) return fail(QTIP_ERR_INVALID_PARAMS, "NULL output");
    if (!hadamard_factor(n, &bb, &aa)) return fail(QTIP_ERR_SHAPE, "no supported Hadamard order");
    *b = bb;
    *a = aa;
    return QTIP_OK;
}

void qtip_set_matvec_impl(int impl) { g_impl = impl; }

void qtip_set_pdl(int enable) { g_pdl = enable != 0; }

void qtip_profile_events(void* ev_start, void* ev_stop) {
    g_prof_start = (cudaEvent_t)ev_start;
    g_prof_stop = (cudaEvent_t)ev_stop;
}
int qtip_get_matvec_impl(void) { return g_impl; }

const char* qtip_status_string(qtip_status s) {
    switch (s) {
        case QTIP_OK: return "QTIP_OK";
        case QTIP_ERR_INVALID_PARAMS: return "QTIP_ERR_INVALID_PARAMS";
        case QTIP_ERR_SHAPE: return "QTIP_ERR_SHAPE";
        case QTIP_ERR_INVALID_PATH: return "QTIP_ERR_INVALID_PATH";
        case QTIP_ERR_ALIGNMENT: return "QTIP_ERR_ALIGNMENT";
        case QTIP_ERR_UNSUPPORTED: return "QTIP_ERR_UNSUPPORTED";
        case QTIP_ERR_CUDA: return "QTIP_ERR_CUDA";
        case QTIP_ERR_WORKSPACE: return "QTIP_ERR_WORKSPACE";
    }
    return "QTIP_ERR_UNKNOWN";
}

const char* qtip_last_error(void) { return g_err.c_str(); }

uint64_t qtip_launch_count(void) { return g_launches; }

}  // extern "C"

// Test / profiling hook: per-CTA timelines of the RHT and mma GEMV kernels into buf (u64, see
// trace.cuh; cap records); buf = NULL turns tracing off.
// Test / tuning knobs: 1 = fused split-K reduction in the mma GEMV (default 0: measured slower,
// DESIGN.md).
extern "C" int qtip_internal_set_knob(int key, int value) {
    if (key == 1) { g_fused_reduce = value != 0; return 0; }
    if (key == 2) { qtip::g_layer_debug = value; return 0; }
    if (key == 3) { g_layer_auto = value != 0; return 0; }
    if (key == 4) { g_l2_prefetch = value; return 0; }
    return -1;
}

extern "C" int qtip_internal_set_layer_trace(void* buf, int cap) {
    return (int)qtip::set_cta_trace_layer((unsigned long long*)buf, cap);
}

extern "C" int qtip_internal_set_cta_trace(void* buf, int cap) {
    cudaError_t e = qtip::set_cta_trace_rht((unsigned long long*)buf, cap);
    if (e == cudaSuccess) e = qtip::set_cta_trace_mma((unsigned long long*)buf, cap);
    if (e == cudaSuccess) e = qtip::set_cta_trace_row((unsigned long long*)buf, cap);
    if (e == cudaSuccess) e = qtip::set_cta_trace_layer((unsigned long long*)buf, cap);
    return (int)e;
}
