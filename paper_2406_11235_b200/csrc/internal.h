// internal.h -- host-side declarations shared by the libqtip translation units.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace qtip {

void count_launch(int n);
int num_sms();
// api.cu's status / message helpers and code arguments, for entry points defined in other files.
qtip_status api_fail(qtip_status s, const char* msg);
qtip_status api_cuda_fail(cudaError_t e, const char* where);
struct CodeArgs;
CodeArgs api_code_args(const qtip_params* p);

// Launch with programmatic dependent launch enabled (the kernel may start while its predecessor
// on the stream drains; it must griddepcontrol.wait before reading the predecessor's output).
// Every libqtip kernel asks for the maximum shared-memory carve-out, so consecutive kernels never
// force an SM re-partition of L1/shared memory between launches.
void prefer_max_smem(const void* kern);
bool pdl_enabled();

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    prefer_max_smem((const void*)kern);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// Cooperative launch (the driver guarantees every CTA of the grid is co-resident, or refuses the
// launch) for kernels that spin on grid-wide barriers / tickets (k_layer.cu): two such grids on
// concurrent streams, or under MPS, could otherwise split the SMs and wait on each other.  PDL is
// kept when enabled.
template <typename... KArgs, typename... Args>
cudaError_t launch_coop(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    prefer_max_smem((const void*)kern);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// Hadamard factor tables (hadamard.cpp): n = b * 2^a; device +-1 table of H_b (or H_b^T), one
// bit row per matrix row padded to 32-bit words (bit j of row i set <=> entry = -1), cached per device.
bool hadamard_factor(int64_t n, int* b, int* a);
const uint32_t* hadamard_table_device(int b, bool transpose, cudaError_t* err);

// Kernel launchers.
cudaError_t launch_decode(const Layout& lay, int code, int V, const CodeArgs& ca, const void* packed,
                          const uint16_t* lut, int out_f32, void* out, cudaStream_t s);

// Largest number of same-shape layers one grouped launch serves (q, k, v / gate, up).
constexpr int kMaxGroup = 4;

struct RhtPlan {
    int64_t n;
    int b, a;          // n = b * 2^a
    int a2;            // Walsh-Hadamard length L2 = 2^a2 done in registers / shuffles
    int f;             // order of the dense factor D = H_b (x) H_{2^(a - a2)}, f = n / L2
    int E;             // columns per lane (L2 / 32, at least 1)
    int RA;            // rows of D accumulated per lane
    int rows_per_cta;  // rows of D per CTA (RA * 32 / min(L2, 32))
    const uint32_t* hb;   // device H_b bit rows (nullptr when b == 1)
    const uint32_t* hbt;  // device H_b^T bit rows (inverse transform)
};
// min_ctas: rows of D per CTA are chosen so that one transform still has >= min_ctas CTAs (a grouped
// launch of G transforms passes 128 / G to stay within one wave).
cudaError_t make_rht_plan(int64_t n, RhtPlan* plan, int min_ctas = 128, int64_t B = 1);
// out[bt][i] = scale * (M v)[i] / sqrt(n) with v = in * s (forward) or in (inverse, then * s).
// in/out batch strides in elements.  out_mode 0 float32, 1 binary16 duplicated per 32-bit word,
// 2 binary16; elements [n, pad_to) of every output row are written as zero.
// zero_ptr[0 .. zero_n) is cleared after the kernel's PDL wait (the GEMV's split-K arrival counters).
cudaError_t launch_rht(const RhtPlan& plan, int64_t B, const uint8_t* sign, const float* in, int64_t in_stride,
                       void* out, int64_t out_stride, int inverse, float scale, cudaStream_t s, int out_mode = 0,
                       int64_t pad_to = 0, int* zero_ptr = nullptr, int zero_n = 0);
// G transforms of the same plan in one launch (grid.z = g): sign[g], in[g], out[g], scale[g];
// zero[g][0 .. zero_n) cleared after the PDL wait (the GEMVs' counters), when zero is given.
cudaError_t launch_rht_group(const RhtPlan& plan, int G, int64_t B, const uint8_t* const* sign, const float* const* in,
                             int64_t in_stride, void* const* out, int64_t out_stride, int inverse, const float* scale,
                             cudaStream_t s, int out_mode = 0, int64_t pad_to = 0, int* const* zero = nullptr,
                             int zero_n = 0);
// The next launch_rht / launch_rht_group on this host thread L2-prefetches bytes[g] from ptr[g]
// (its transform g) before its PDL wait: the weights of the GEMV that follows it.
void rht_set_prefetch(int G, const void* const* ptr, const uint64_t* bytes);
// x (float32) -> out_mode encoding, zero padded to pad_to (used when RHT-in is off).
cudaError_t launch_convert(const float* in, int64_t n, int64_t in_stride, int64_t B, void* out, int64_t out_stride,
                           int out_mode, int64_t pad_to, cudaStream_t s, int* zero_ptr = nullptr, int zero_n = 0);

// Reference (CUDA-core) fused decode-GEMV: partial[kc][b][row] over the row blocks [rb0, rb1).
cudaError_t launch_gemv_simple(const Layout& lay, int code, const CodeArgs& ca, const void* packed,
                               const uint16_t* lut, const float* xt, int64_t B, int64_t rb0, int64_t rb1,
                               float* partial, cudaStream_t s);
// tcgen05 fused decode-GEMM (k_gemv_tc.cu); x~ in the compact binary16 encoding of
// gemv_tc_xt_mode(code) with row stride xt_row_bytes.
bool gemv_tc_supported(const Layout& lay, int code, const CodeArgs& ca, int64_t B);
int gemv_tc_xt_mode(int code);
cudaError_t launch_gemv_tc(const Layout& lay, int code, const CodeArgs& ca, const void* packed, const uint16_t* lut,
                           const void* xt_compact, int64_t xt_row_bytes, int64_t B, int64_t rb0, int64_t rb1,
                           float* partial, cudaStream_t s);
// Register-fed mma.sync fused decode-GEMV (k_gemv_mma.cu); same x~ encoding as the tcgen05 kernel.
// x~ in fragment order (out_mode gemv_mma_xt_mode(code)), gemv_mma_batch_pad(B) rows of
// xt_row_words 32-bit words (rows >= B may hold anything: they only feed discarded columns).
bool gemv_mma_supported(const Layout& lay, int code, const CodeArgs& ca, int64_t B);
int gemv_mma_xt_mode(int code);
int gemv_mma_batch_pad(int64_t B);
// Split-K reduction fused in: the last CTA to finish a row block (arrival counter cnt[RB], zero
// on entry and left zero) writes y[b][i - row_lo] = scale * sum_kc partial[kc][b][i] for the
// block's rows i in [row_lo, row_hi), in launch_reduce's association (bitwise equal to it).
struct MmaEpilogue {
    int* cnt;          // n_rb arrival counters, then the work counter (all zero on entry)
    int64_t n_rb;
    float* y;
    int64_t y_stride;
    int64_t row_lo, row_hi;
    float scale;
};
cudaError_t launch_gemv_mma(const Layout& lay, int code, const CodeArgs& ca, const void* packed, const uint16_t* lut,
                            const void* xt_frag, int64_t xt_row_words, int64_t B, int64_t rb0, int64_t rb1,
                            float* partial, const MmaEpilogue& ep, cudaStream_t s);
// y[b][i - row0] = scale * sum_kc partial[kc][b][i] for rows [row0, row1).
cudaError_t launch_reduce(const float* partial, int64_t n_kc, int64_t B, int64_t m_pad, int64_t row0, int64_t row1,
                          float scale, float* y, int64_t y_stride, cudaStream_t s);

// Row-tile fused decode-GEMV (k_gemv_row.cu, impl 4): one CTA per tile row, no split-K; writes
// y[b * y_stride + (i - row_lo)] = scale * (W~ x~)[i] for rows i in [row_lo, row_hi).
bool gemv_row_supported(const Layout& lay, int code, const CodeArgs& ca, int64_t B);
cudaError_t launch_gemv_row(const Layout& lay, int code, const CodeArgs& ca, const void* packed, const uint16_t* lut,
                            const void* xt_frag, int64_t xt_row_words, int64_t B, int64_t row_begin, int64_t row_end,
                            float* y, int64_t y_stride, int64_t row_lo, int64_t row_hi, float scale, cudaStream_t s);

// Fused single-launch layer (k_layer.cu, impl 5): RHT-in, decode-GEMV, reduction and RHT-out with
// in-kernel grid barriers (one CTA per SM).  ws_f: layer_workspace_floats() floats; bar: 256
// per-CTA epoch flags that must be zero before the first call (every call leaves them equal).
bool layer_supported(const Layout& lay, int code, const CodeArgs& ca, int64_t B, int64_t tile_rows, bool rht_in,
                     bool rht_out);
size_t layer_workspace_floats(const Layout& lay, int64_t B, int64_t tile_rows);
cudaError_t launch_layer(const Layout& lay, int code, const CodeArgs& ca, const void* packed, const uint16_t* lut,
                         const float* x, const uint8_t* sign_n, const uint8_t* sign_m, float scale, float* y,
                         int64_t B, int64_t row_begin, int64_t row_end, bool rht_in, bool rht_out, bool xt_ready,
                         uint32_t* xt_g, int64_t row_words, float* ws_f, unsigned* bar, cudaStream_t s);
// G same-shape layers in one persistent launch (x~ already in each layer's workspace, no RHT
// phases): CTAs [g P / G, (g+1) P / G) run layer g in rows mode.  cudaErrorInvalidConfiguration
// when a layer has fewer tile rows than its CTAs or the shared memory does not fit.
bool layer_group_supported(const Layout& lay, int code, const CodeArgs& ca, int64_t B, int G);
cudaError_t launch_layer_group(const Layout& lay, int code, const CodeArgs& ca, int G, const void* const* packed,
                               const uint16_t* const* lut, const float* scale, float* const* y, int64_t B,
                               uint32_t* const* xt_g, int64_t row_words, float* const* ws_f, unsigned* const* bar,
                               cudaStream_t s);

// tcgen05 stream-K fused decode-GEMV (k_umma.cu, impl 7): G same-shape layers' row blocks
// [rb0, rb1), x~ per layer in the UMMA B layout (RHT out_mode umma_xt_mode(code), batch stride
// umma_batch_pad(B)).  Writes yout[g][b * ys + i] = yscale[g] * (W~ x~)[i] for launch rows i in
// [0, rows); seg[g] (umma_seg_floats floats) holds partial sums of split row blocks, ticket[g]
// (rb1 - rb0 ints, zero on entry and left zero) their arrival counters.  HYB layers of a group share
// one LUT.
bool umma_supported(const Layout& lay, int code, const CodeArgs& ca, int64_t B, int G);
int umma_xt_mode(int code);
int umma_batch_pad(int64_t B);
size_t umma_seg_floats(const Layout& lay, int code, int64_t B);
cudaError_t launch_umma(const Layout& lay, int code, const CodeArgs& ca, int G, const void* const* packed,
                        const uint16_t* lut, const void* const* xt, float* const* seg, int* const* ticket,
                        float* const* yout, const float* yscale, int64_t ys, int64_t rows, int64_t B, int64_t rb0,
                        int64_t rb1, cudaStream_t s);

// The code variants of NEXT-3 (k_variant.cu): the lookup-only code and HYB with V = 1.  Decode, and
// the fused decode-GEMV partial[kc][b][row] over row blocks [rb0, rb1) with x~ float32 (row stride
// n_pad); the whole table is staged in shared memory (variant_gemv_smem bytes).
bool is_variant(const qtip_params* p);
cudaError_t launch_variant_decode(const qtip_params* p, const Layout& lay, const void* packed, const uint16_t* lut,
                                  int out_f32, void* out, cudaStream_t s);
cudaError_t launch_variant_gemv(const qtip_params* p, const Layout& lay, const void* packed, const uint16_t* lut,
                                const float* xt, int64_t B, int64_t rb0, int64_t rb1, float* partial, cudaStream_t s);
size_t variant_gemv_smem(const qtip_params* p, int64_t B);

// Tail-biting trellis quantizer (k_viterbi.cu): Algorithm 4 per sequence of T source values (in
// code units), binary32 DP.  ws: viterbi_workspace_bytes(T) bytes (backpointers, per CTA).
bool viterbi_supported(int code, int k, int V, int L, int Q, int two_sign);
size_t viterbi_workspace_bytes(int T);
// The sequences of a matrix (T_x x T_y blocks in row-major scan, scaled): out[(I n/T_y + J) T + p].
cudaError_t launch_gather_sequences(const float* W, int64_t m, int64_t n, int Tx, int Ty, float scale, float* out,
                                    cudaStream_t s);
cudaError_t launch_viterbi(int code, int kv, const CodeArgs& ca, const float* src, const uint16_t* lut, int nseq, int T,
                           uint32_t* states, float* cost, void* ws, cudaStream_t s);

// Debug CTA timelines (trace.cuh), per translation unit.
cudaError_t set_cta_trace_rht(unsigned long long* buf, int cap);
cudaError_t set_cta_trace_mma(unsigned long long* buf, int cap);
cudaError_t set_cta_trace_row(unsigned long long* buf, int cap);
cudaError_t set_cta_trace_layer(unsigned long long* buf, int cap);
extern int g_layer_debug;   // k_layer.cu debug bits (qtip_internal_set_knob(2, bits))

}  // namespace qtip
