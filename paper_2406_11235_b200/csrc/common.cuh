// common.cuh -- device layout and shared definitions of libqtip (sm_100a).
//
// Device layout of a packed m x n matrix (private to the library, produced by qtip_pack):
//   * tile (16 x 16 weights, one T = 256 trellis sequence) = TW = 8k
//     32-bit words; word w holds logical stream bits [32w, 32w+32) MSB-first, so bit 31
//     of word w is stream bit 32w.
//   * cell = 8 tile-rows x 8 tile-columns (128 output rows x 128 input columns), the unit
//     of work of the GEMV kernels and one contiguous 2048k-byte block (one bulk copy).
//     Cells are stored row-block major: cell (RB, KC) at word (RB * NKC + KC) * CELL_WORDS.
//   * inside a cell the two tiles of a column pair (J = 2p, 2p+1) are word-interleaved:
//       word(I, J, w) = ((I * 4 + J/2) * TW + w) * 2 + (J & 1)
//     so the thread that owns output row r of both tiles fetches (tile 2p, tile 2p+1) word
//     w with one 64-bit load.
//   * rows and columns are padded to multiples of 128 with zero tiles; the padded
//     activations are zero, so padding never changes a result.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#include "../../include/qtip.h"

namespace qtip {

constexpr int kTile = 16;
constexpr int kCellTileRows = 8;
constexpr int kCellTileCols = 8;
constexpr int kCellRows = kTile * kCellTileRows;   // 128
constexpr int kCellCols = kTile * kCellTileCols;   // 128

struct Layout {
    int64_t m, n;          // logical shape
    int64_t m_pad, n_pad;  // padded to 128
    int64_t n_rb, n_kc;    // cells along rows / columns
    int k;
    int tw;                // words per tile = 8k
    int64_t cell_words;    // 128 * tw
};

inline Layout make_layout(int64_t m, int64_t n, int k) {
    Layout l;
    l.m = m; l.n = n; l.k = k;
    l.m_pad = (m + kCellRows - 1) / kCellRows * kCellRows;
    l.n_pad = (n + kCellCols - 1) / kCellCols * kCellCols;
    l.n_rb = l.m_pad / kCellRows;
    l.n_kc = l.n_pad / kCellCols;
    l.tw = 8 * k;
    l.cell_words = (int64_t)kCellTileRows * kCellTileCols * l.tw;
    return l;
}

__host__ __device__ inline int64_t cell_word_index(int I, int J, int w, int tw) {
    return ((int64_t)(I * 4 + (J >> 1)) * tw + w) * 2 + (J & 1);
}

// Code parameters as the kernels see them.
struct CodeArgs {
    uint32_t a, b;        // LCG
    uint32_t magic;       // 3INST: (m << 16) | m
    int Q;
    int two_sign;
};

}  // namespace qtip
