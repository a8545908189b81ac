/* qtip.h -- C ABI of libqtip, the B200 (sm_100a) QTIP inference library.
 *
 * QTIP (arXiv 2406.11235) stores an RHT-processed weight matrix W~ (m x n) as 16 x 16
 * tiles, each tile one T = 256 sequence (row-major scan)
 * tail-biting-quantized on an (L, k, V) bitshift trellis (PAPER.md:121-125, :207-214,
 * :325-328) and decoded by a computed code (1MAD Alg. 1 :269-281, 3INST Alg. 2 :283-296)
 * or the hybrid lookup code (HYB Alg. 3 :311-321).  Inference computes
 *
 *     y = scale * S_m H_m^T W~ H_n S_n x                 (RHT)
 *
 * where H_k is an orthonormal Hadamard matrix (reading R7: kron(Paley-I H_b,
 * Sylvester H_{2^a}), b the smallest supported order with k/b a power of two) and
 * S_k a random sign vector.
 *
 * Conventions for every call:
 *   - "d_" pointers are DEVICE pointers, "h_" pointers HOST pointers.  The caller owns
 *     every buffer; the library never frees caller memory.  The only memory the library
 *     allocates itself is a per-device cache of constant Hadamard +-1 tables (a few KB),
 *     created on first use and kept for the process lifetime.
 *   - stream is a cudaStream_t passed as void* (NULL = legacy default stream).  Device
 *     work is enqueued on it asynchronously; host-side validation happens before any
 *     launch, so a non-OK status means nothing was enqueued (except QTIP_ERR_CUDA).
 *   - Shapes: m, n multiples of 16 (one tile).  Batch B >= 1.
 *   - Errors are returned by value; qtip_last_error() gives a thread-local detail string.
 *   - Logical tile stream: kT bits, MSB-first (bit 0 = most significant bit of byte 0),
 *     tiles ordered [m/16][n/16]; state t of a tile is the L-bit window at bit t*kV,
 *     wrapping mod kT (tail-biting).  This is the format the oracle and SPEC use; the
 *     DEVICE layout ("packed") is private to the library and produced by qtip_pack*.
 */
#ifndef QTIP_H_
#define QTIP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    QTIP_OK = 0,
    QTIP_ERR_INVALID_PARAMS = -1, /* unsupported (L,k,V,code,Q), NULL pointer, bad flags   */
    QTIP_ERR_SHAPE = -2,          /* m/n not multiples of 16, no Hadamard order, bad rows    */
    QTIP_ERR_INVALID_PATH = -3,   /* qtip_pack_states: edge rule or tail-biting closure fails */
    QTIP_ERR_ALIGNMENT = -4,      /* a device pointer is not 16-byte aligned                 */
    QTIP_ERR_UNSUPPORTED = -5,    /* valid QTIP parameters this build has no kernel for      */
    QTIP_ERR_CUDA = -6,           /* a CUDA call failed (detail in qtip_last_error)          */
    QTIP_ERR_WORKSPACE = -7       /* workspace too small (see qtip_matvec_workspace_bytes)   */
} qtip_status;

/* QTIP_CODE_LUT: the lookup-only code: value of state x = LUT[x], a 2^L-entry
 * binary16 table (L = 14: 32 KB), V = 1, blocks T_x x T_y = 32 x 8 or 16 x 16. */
typedef enum { QTIP_CODE_1MAD = 1, QTIP_CODE_3INST = 2, QTIP_CODE_HYB = 3, QTIP_CODE_LUT = 4 } qtip_code;

/* Trellis + code parameters (PAPER.md:121 (L,k,V); :260, :267 LCG constants; :303 Q). */
typedef struct {
    int32_t L;            /* state bits: 16; the LUT code takes kV <= L <= 16 (14) */
    int32_t k;            /* bits per weight, 1..4 (device path: 2, 3, 4)                         */
    int32_t V;            /* values per trellis step: 1 for 1MAD/3INST/LUT; HYB 2, or 1 with a 1-D  */
                          /* codebook (Q = 6, V = 1)                                    */
    int32_t code;         /* qtip_code                                                            */
    int32_t Q;            /* HYB LUT index bits; 9 -> 2 KiB table; V = 1: 1..14    */
    int32_t tail_biting;  /* must be 1: kT bits per tile                              */
    int32_t Tx, Ty;       /* 16, 16 (T = 256, one 16x16 tile per sequence); the LUT code */
                          /* also 32, 8; m must then be a multiple of 32               */
    uint32_t lcg_a;       /* 1MAD: 34038481; 3INST: 89226354                      */
    uint32_t lcg_b;       /* 1MAD: 76625530;         3INST: 64248484                              */
    uint32_t m_fp16;      /* 3INST magic m as binary16 bits: 0x3B60 = fp16(0.922)  */
    int32_t hyb_two_sign; /* HYB: also XOR bit 31; default 0 (the paper's numbers)    */
} qtip_params;

/* Fill *p with the paper's defaults for `code` at k bits (L=16, V=1 or 2, Q=9, T=16x16; the LUT
 * code: L = 14, V = 1, T = 32x8). */
void qtip_params_default(qtip_params* p, int32_t code, int32_t k);

/* Validate *p for the device path.  QTIP_OK or QTIP_ERR_INVALID_PARAMS/UNSUPPORTED. */
qtip_status qtip_params_check(const qtip_params* p);

/* Bytes of the device layout for an m x n matrix (rows and columns padded to 128;
 * padding tiles are zero and multiply zero activations).  Returns -1 on bad params. */
int64_t qtip_packed_bytes(const qtip_params* p, int64_t m, int64_t n);

/* Lay out logical tile streams in device format.
 *   h_tiles: HOST uint8[m/16][n/16][k*T/8] (k*32 bytes per tile), MSB-first, tail-biting.
 *   d_packed: DEVICE buffer of qtip_packed_bytes(p, m, n) bytes, 16-byte aligned.
 * Any bit string is a valid tail-biting walk, so no path validation happens.
 * Synchronous with respect to h_tiles: returns after the copy to d_packed completed. */
qtip_status qtip_pack(const qtip_params* p, int64_t m, int64_t n, const uint8_t* h_tiles,
                      void* d_packed, void* stream);

/* As qtip_pack, from state walks (SPEC pack(path)): h_states HOST uint32[m/16][n/16][T/V].
 * Every consecutive pair must satisfy the edge rule and the last state must
 * connect to the first (tail-biting closure), else QTIP_ERR_INVALID_PATH. */
qtip_status qtip_pack_states(const qtip_params* p, int64_t m, int64_t n, const uint32_t* h_states,
                             void* d_packed, void* stream);

/* Dense RHT-domain weights W~ (raw code values, no scale; P:123 reconstruction).
 *   d_lut: HYB, DEVICE uint16[2^Q][2] binary16 (c0, c1) pairs; HYB with V = 1: uint16[2^Q];
 *     the LUT code: uint16[2^L]; NULL for 1MAD/3INST.  (16-byte aligned for the matvec.)
 *   out_dtype 0: binary16 (normative, bit-exact vs the oracle); 1: float32 = exact widening.
 *   d_out: DEVICE [m][n] row-major. */
qtip_status qtip_decode(const qtip_params* p, int64_t m, int64_t n, const void* d_packed,
                        const uint16_t* d_lut, int out_dtype, void* d_out, void* stream);

#define QTIP_RHT_IN  1  /* apply x~ = H_n S_n x / sqrt(n) before the product               */
#define QTIP_RHT_OUT 2  /* apply y = S_m H_m^T y~ / sqrt(m) after it (needs all m rows)    */
#define QTIP_XT_READY 4 /* kernel benchmarking: reuse the x~ left in d_workspace by the previous
                           call with the same (p, m, n, B, workspace) instead of transforming
                           d_x again (d_x and d_sign_n are then ignored)                     */

/* Fused decode + matrix-vector product, batch B (<= 64):
 *     d_y[b][i - row_begin] = scale * (S_m H_m^T W~ H_n S_n x_b)[i],  i in [row_begin, row_end)
 *   d_x: DEVICE float32 [B][n];  d_y: DEVICE float32 [B][row_end - row_begin].
 *   d_sign_n / d_sign_m: DEVICE bit-packed signs (element i negative iff bit (i&7) of byte
 *     i>>3 is set), ceil(n/8) / ceil(m/8) bytes; ignored when the matching flag is off.
 *   flags: QTIP_RHT_IN | QTIP_RHT_OUT (| QTIP_XT_READY).  Without RHT_OUT the result is
 *     scale * W~ x~.
 *     A partial row range (row_begin > 0 or row_end < m) requires RHT_OUT off; row_begin
 *     and row_end must be multiples of 128 (or row_end == m).
 *   d_workspace: DEVICE scratch of >= qtip_matvec_workspace_bytes(...) bytes, 256-B aligned,
 *     zero-filled before its first use.  It holds x~, partial sums and the kernels' arrival
 *     counters / grid-barrier words: every call leaves those counters zero (or, for the grid
 *     barriers, in a consistent state), and every call that transforms x (no QTIP_XT_READY)
 *     clears them before the GEMV starts, so only a QTIP_XT_READY call on never-used scratch
 *     needs the zero fill.  Not shared between concurrent calls.
 *   Deterministic: the reduction order depends on (p, m, n, B, row range, SM count), never on
 *     timing -- repeated calls are bitwise identical.  Kernels 1-6 split K by (m, n) only, so a
 *     row shard reproduces the full call's rows bit for bit; the stream-K kernel (7) cuts the
 *     launch's own cells into equal ranges, so a shard's rows agree with the full call only to
 *     fp32 rounding (both within the 1e-3 parity bar).
 *   The kernel choice (auto) depends on (p, m, n, B) only, not on the row range, so QTIP_XT_READY
 *     reuses an x~ written by a call with any row range. */
qtip_status qtip_matvec(const qtip_params* p, int64_t m, int64_t n, int64_t B,
                        const void* d_packed, const uint16_t* d_lut,
                        const uint8_t* d_sign_n, const uint8_t* d_sign_m, float scale,
                        const float* d_x, float* d_y, int64_t row_begin, int64_t row_end,
                        int flags, void* d_workspace, size_t workspace_bytes, void* stream);

size_t qtip_matvec_workspace_bytes(const qtip_params* p, int64_t m, int64_t n, int64_t B);

/* G (1..4) layers of the SAME shape (m, n) and parameters applied to the SAME input x, e.g. the
 * q, k, v projections or gate, up of a transformer block (QTIP quantizes q, k, v, o, up,
 * gate, down as 7 separate matrices, each with its own RHT signs):
 *     d_y[g] = qtip_matvec(p, m, n, B, d_packed[g], d_lut[g], d_sign_n[g], d_sign_m[g], scale[g],
 *                          d_x, d_y[g], 0, m, flags, d_workspace[g], ...)
 *   Arrays of G HOST pointers to DEVICE buffers (d_packed, d_lut (NULL array unless HYB),
 *   d_sign_n, d_sign_m, d_y, d_workspace); scale: HOST float[G]; each workspace >= qtip_matvec_workspace_bytes(p, m, n, B)
 *   (workspace_bytes is the size of each), 256-B aligned.  Full row range only.
 *   When the persistent kernel fits (B <= 4, every layer keeps >= 1 tile row per CTA) the G
 *   layers run as ONE grouped RHT-in launch, ONE persistent decode-GEMV launch (the SMs split
 *   between the layers) and ONE grouped RHT-out launch; otherwise G qtip_matvec calls.  Results
 *   equal G qtip_matvec calls with qtip_set_matvec_impl(6) bit for bit (canonical row sums, R18).
 *   Errors as qtip_matvec, plus QTIP_ERR_INVALID_PARAMS for G outside 1..4 or NULL arrays. */
/* 1 if qtip_matvec_group with these arguments runs as the grouped launches (else G per-layer calls,
 * which a caller may prefer to run concurrently on its own streams), 0 otherwise. */
int qtip_matvec_group_fused(const qtip_params* p, int G, int64_t m, int64_t n, int64_t B);

qtip_status qtip_matvec_group(const qtip_params* p, int G, int64_t m, int64_t n, int64_t B,
                              const void* const* d_packed, const uint16_t* const* d_lut, const uint8_t* const* d_sign_n,
                              const uint8_t* const* d_sign_m, const float* scale, const float* d_x, float* const* d_y,
                              int flags, void* const* d_workspace, size_t workspace_bytes, void* stream);

/* A CHAIN of dependent layers in one persistent launch (impl 8, k_chain.cu): a decode step of a
 * model applies its linear layers in stages, each stage's layers reading one input that is the
 * output of a layer of the previous stage (q, k, v -> o -> gate, up -> down -> next q, k, v):
 *     stage 0:  d_y[l] = scale_l S_m H_m^T W~_l H_n S_n x
 *     stage s:  the same with x := d_y[src_l], src_l a layer of stage s-1
 * i.e. exactly the qtip_matvec calls (RHT in and out) made one after another, but with the weight
 * stream and trellis decode of later layers overlapping the transforms and hand-offs of earlier
 * ones (no kernel boundary between layers).
 *   layers: HOST array in stage order; stage numbers 0, 1, 2, ... (consecutive, non-decreasing);
 *     the layers of one stage share n and src; stage 0 has src = -1 (the external x); a stage
 *     holds 1..4 layers; src's m must equal the reader's n.  d_packed (16-B aligned, qtip_pack
 *     layout), d_sign_n / d_sign_m (as qtip_matvec) and d_y (DEVICE float32 [B][m], written by
 *     every run) are the caller's and must stay valid while the plan is used.
 *   p: as qtip_matvec with 2 <= k <= 4; HYB needs Q = 9, one-sign and d_lut (one table for every
 *     layer of the chain).  B: 1..16.  m, n: multiples of 16 with a supported Hadamard order.
 *   qtip_chain_plan_create validates, builds the device tables and allocates the plan's own device
 *     memory (x~ / y~ / partial-sum buffers and counters, ~(n + 4m + 512 (P + m/128)) B bytes per
 *     layer, P = SM count) on the current device; it synchronises the device once.  Errors:
 *     QTIP_ERR_INVALID_PARAMS (structure), QTIP_ERR_SHAPE, QTIP_ERR_ALIGNMENT, QTIP_ERR_UNSUPPORTED
 *     (batch, code, stage too large, shared memory), QTIP_ERR_CUDA.
 *   qtip_chain_run: d_x DEVICE float32 [B][n of stage 0]; stream-ordered, graph-capturable (a
 *     memset of the plan's counters, then one cooperative kernel).  One run at a time per plan.
 *   Results: every layer's y within the qtip_matvec parity bar of the float64 definition applied
 *     to that layer's actual input; deterministic for a given plan and SM count.
 *   qtip_chain_plan_destroy frees the plan (NULL is a no-op). */
typedef struct {
    const void* d_packed;
    const uint8_t* d_sign_n;
    const uint8_t* d_sign_m;
    float scale;
    int64_t m, n;
    float* d_y;
    int32_t stage;
    int32_t src;
} qtip_chain_layer;
typedef struct qtip_chain_plan qtip_chain_plan;
qtip_status qtip_chain_plan_create(const qtip_params* p, int32_t nlayers, const qtip_chain_layer* layers, int64_t B,
                                   const uint16_t* d_lut, qtip_chain_plan** plan);
qtip_status qtip_chain_run(qtip_chain_plan* plan, const float* d_x, void* stream);
void qtip_chain_plan_destroy(qtip_chain_plan* plan);
int32_t qtip_chain_plan_stages(const qtip_chain_plan* plan);

/* Random Hadamard transform of B vectors of length n:
 *   inverse = 0:  out = H_n (S . in) / sqrt(n)
 *   inverse = 1:  out = S . (H_n^T in) / sqrt(n)
 * d_in, d_out: DEVICE float32 [B][n], distinct buffers (out-of-place; d_in == d_out is
 * QTIP_ERR_INVALID_PARAMS). */
qtip_status qtip_rht(int64_t n, int64_t B, const uint8_t* d_sign, const float* d_in, float* d_out,
                     int inverse, void* stream);

/* The Hadamard factorisation used for order n: n = b * 2^a.  QTIP_ERR_SHAPE if none. */
qtip_status qtip_hadamard_order(int64_t n, int32_t* b, int32_t* a);

/* Tail-biting trellis quantizer (P:127-141 Viterbi DP; Algorithm 4): for each of nseq
 * independent length-T source sequences, the walk returned by Algorithm 4 -- rotate the sequence
 * right by floor(T/2), run the unconstrained Viterbi, take the L-kV bit overlap O at the seam
 * (reading R3: bottom L-kV bits of the rotated walk's state at 1-indexed group floor(T/(2V))),
 * then run the Viterbi on the original sequence with the first state's top and the last state's
 * bottom L-kV bits both equal to O (a tail-biting walk).
 *   p: L = 16 and either 3INST/1MAD with V = 1, k in {2, 3, 4}, or HYB with V = 2, k in {2, 3, 4},
 *     Q = 9, one-sign (else QTIP_ERR_UNSUPPORTED).  T % V == 0.
 *   d_source: DEVICE float32 [nseq][T], already in code units (the caller scales the source by
 *     the code's state standard deviation, reading R9); d_lut: HYB table as for qtip_decode (DEVICE
 *     binary16 pairs (c0, c1) [2^Q][2]), NULL otherwise; d_states: DEVICE uint32 [nseq][T/V] walk
 *     (feed to qtip_pack_states after copying to the host); d_cost: DEVICE float32 [nseq], the
 *     walk's squared error sum.
 *   Arithmetic: code values are the binary16 codes of qtip_decode widened to binary32; the DP
 *     is binary32 with each operation rounded separately (per step sum_v (c_v - s_v)^2 left to
 *     right), ties to the smallest predecessor index and the smallest final state (reading R4), as
 *     oracle/viterbi.c qo_viterbi_f32 (R17).
 *   d_workspace: qtip_viterbi_workspace_bytes(p, T) bytes, caller-owned (backpointers). */
size_t qtip_viterbi_workspace_bytes(const qtip_params* p, int64_t T);
qtip_status qtip_viterbi_tailbite(const qtip_params* p, int64_t nseq, int64_t T, const float* d_source,
                                  const uint16_t* d_lut, uint32_t* d_states, float* d_cost, void* d_workspace,
                                  size_t workspace_bytes, void* stream);

/* Quantize a whole RHT-domain matrix (the step before qtip_pack_states): every T_x x T_y block of
 * d_W is one sequence in row-major scan, multiplied by source_scale (reading R9:
 * the code's state standard deviation, so the source is in code units), then Algorithm 4 as
 * qtip_viterbi_tailbite (same support, same binary32 arithmetic).
 *   d_W: DEVICE float32 [m][n]; d_states: DEVICE uint32 [m/T_x][n/T_y][T/V] (the layout
 *   qtip_pack_states reads after a copy to the host); d_cost: DEVICE float32 [m/T_x][n/T_y];
 *   d_workspace: qtip_quantize_workspace_bytes(p, m, n) bytes, caller-owned. */
size_t qtip_quantize_workspace_bytes(const qtip_params* p, int64_t m, int64_t n);
qtip_status qtip_quantize_matrix(const qtip_params* p, int64_t m, int64_t n, const float* d_W, float source_scale,
                                 const uint16_t* d_lut, uint32_t* d_states, float* d_cost, void* d_workspace,
                                 size_t workspace_bytes, void* stream);

/* Selects the matvec kernel: 0 = auto (the measured-fastest supported kernel), 1 = CUDA-core
 * reference kernel, 2 = tcgen05 kernel (A in TMEM, per-cell split-K), 3 = register-fed mma.sync
 * kernel with split-K over 128-column cells, 4 = row-tile mma.sync kernel (one CTA per 16 rows,
 * B <= 4), 5 = fused single-launch layer kernel (RHT-in, GEMV, RHT-out with in-kernel grid
 * barriers), 6 = RHT kernels around the persistent row-owning GEMV of 5, 7 = RHT kernels around the
 * stream-K tcgen05 GEMV (k_umma.cu: decoded binary16 weights in TMEM, asynchronous UMMA, equal
 * cell ranges per SM, one x~ slab per cell; auto for HYB at every batch with >= 10 cells per SM,
 * for 3INST with >= 20 cells per SM below batch 8 and at every size from batch 8, for 1MAD with >= 40).
 * Process-wide; for ablations and tests. */
void qtip_set_matvec_impl(int impl);
int qtip_get_matvec_impl(void);

/* Bench instrumentation: arms the NEXT qtip_matvec call on this thread to record the two
 * cudaEvent_t handles (passed as void*) on its stream immediately before and after its fused
 * decode-GEMV kernel, then disarms.  NULL, NULL disarms explicitly. */
void qtip_profile_events(void* ev_start, void* ev_stop);

/* Programmatic dependent launch between the library's kernels (default on).  Off isolates
 * each kernel's duration for measurement. */
void qtip_set_pdl(int enable);

const char* qtip_status_string(qtip_status s);
const char* qtip_last_error(void);
/* Number of kernels this thread has launched through the API (for bench accounting). */
uint64_t qtip_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* QTIP_H_ */
