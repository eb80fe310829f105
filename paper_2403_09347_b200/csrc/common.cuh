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

// Block-sparse grid (BlockGrid, masking.py:33-63, 120-128): is the cell of
// (query position qp, key position kp) skipped?
// Cell indices are clamped: zero-padded rows (positions >= the real length the grid
// tiles) read the last cell; their results are discarded by the caller.
__device__ __forceinline__ int64_t grid_qc(const burst_hop& h, int64_t qp) {
  const int64_t c = qp / h.grid_qcell;
  return c < h.grid_nqb ? c : h.grid_nqb - 1;
}
__device__ __forceinline__ int64_t grid_kc(const burst_hop& h, int64_t kp) {
  const int64_t c = kp / h.grid_kcell;
  return c < h.grid_nkb ? c : h.grid_nkb - 1;
}
__device__ __forceinline__ bool grid_skipped(const burst_hop& h, int64_t qp, int64_t kp) {
  return h.grid_skip[grid_qc(h, qp) * h.grid_nkb + grid_kc(h, kp)] != 0;
}

// Grid-mask bits of a run of `n` (<= 64) consecutive local key rows [k0, k0+n) for one
// query position: bit i set = key k0+i hidden.  One table lookup when the run stays in
// one key cell (the common case), per key otherwise.
__device__ __forceinline__ uint64_t grid_key_bits(const burst_hop& h, int64_t qp, int64_t k0, int n) {
  const int64_t row = grid_qc(h, qp) * h.grid_nkb;
  const int64_t kp0 = pos_of(h.k_map, k0), kp1 = pos_of(h.k_map, k0 + n - 1);
  if (kp1 - kp0 == n - 1 && grid_kc(h, kp0) == grid_kc(h, kp1))
    return h.grid_skip[row + grid_kc(h, kp0)] ? (n == 64 ? ~0ull : ((1ull << n) - 1)) : 0ull;
  uint64_t bits = 0;
  for (int i = 0; i < n; ++i)
    if (h.grid_skip[row + grid_kc(h, pos_of(h.k_map, k0 + i))]) bits |= 1ull << i;
  return bits;
}

// Same for a run of `n` (<= 64) consecutive local query rows against one key position.
__device__ __forceinline__ uint64_t grid_query_bits(const burst_hop& h, int64_t q0, int n, int64_t kp) {
  const int64_t col = grid_kc(h, kp);
  const int64_t qp0 = pos_of(h.q_map, q0), qp1 = pos_of(h.q_map, q0 + n - 1);
  if (qp1 - qp0 == n - 1 && grid_qc(h, qp0) == grid_qc(h, qp1))
    return h.grid_skip[grid_qc(h, qp0) * h.grid_nkb + col] ? (n == 64 ? ~0ull : ((1ull << n) - 1))
                                                          : 0ull;
  uint64_t bits = 0;
  for (int i = 0; i < n; ++i)
    if (h.grid_skip[grid_qc(h, pos_of(h.q_map, q0 + i)) * h.grid_nkb + col]) bits |= 1ull << i;
  return bits;
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
