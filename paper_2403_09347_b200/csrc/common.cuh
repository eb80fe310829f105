// Shared device-side definitions: hop geometry, global-position maps, and the
// tile-interleaved ("TL") layout of the fp32 workspaces.
#pragma once
#include <cstdint>
#include "../../include/burst_b200.h"

namespace burst {

// Global position of local row i under a two-segment monotone map
// (contiguous shard: one segment; zigzag shard: chunks i and 2G-1-i).
__host__ __device__ __forceinline__ int64_t pos_of(const burst_posmap& m, int64_t i) {
  return i < m.seg_len ? m.pos0 + i : m.pos1 + (i - m.seg_len);
}

// Number of local rows in [0, n) whose global position is <= p.  Because the
// map is monotone, the causal rule key_pos <= query_pos (masking.py:116-117)
// admits exactly a prefix of the local keys: [0, count_le).
__host__ __device__ __forceinline__ int64_t count_le(const burst_posmap& m, int64_t n, int64_t p) {
  if (p < m.pos0) return 0;
  int64_t c = p - m.pos0 + 1;
  if (c <= m.seg_len) return c < n ? c : n;
  c = m.seg_len;
  if (p >= m.pos1) c += p - m.pos1 + 1;
  return c < n ? c : n;
}

// Tile-interleaved fp32 workspace layout (O_acc, dQ_acc, dK/dV contributions):
// [B*H][ceil(n/128)][D/4][128 rows][4 cols].  A warp whose lanes own 32
// consecutive rows touches one contiguous 512 B run per float4 column group,
// so the thread-per-row TMEM epilogue is fully coalesced.
__host__ __device__ __forceinline__ size_t tl_index(int64_t bh, int64_t row, int col, int D,
                                                    int64_t NT) {
  return ((((size_t)bh * NT + (row >> 7)) * (D >> 2) + (col >> 2)) * 128 + (row & 127)) * 4 +
         (col & 3);
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

}  // namespace burst
