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

// Block-sparse grid (BlockGrid, masking.py:33-63, 120-128).  Global positions and
// cell extents fit in 32 bits (checked on the host), so cell indices use 32-bit
// unsigned division (64-bit division is a long software sequence on the GPU).
// Cell indices are clamped: zero-padded rows (positions >= the real length the grid
// tiles) read the last cell; their results are discarded by the caller.
__device__ __forceinline__ uint32_t grid_qc(const burst_hop& h, int64_t qp) {
  const uint32_t c = (uint32_t)qp / (uint32_t)h.grid_qcell;
  return c < (uint32_t)h.grid_nqb ? c : (uint32_t)h.grid_nqb - 1;
}
__device__ __forceinline__ uint32_t grid_kc(const burst_hop& h, int64_t kp) {
  const uint32_t c = (uint32_t)kp / (uint32_t)h.grid_kcell;
  return c < (uint32_t)h.grid_nkb ? c : (uint32_t)h.grid_nkb - 1;
}
__device__ __forceinline__ bool grid_skipped(const burst_hop& h, int64_t qp, int64_t kp) {
  return h.grid_skip[grid_qc(h, qp) * (uint32_t)h.grid_nkb + grid_kc(h, kp)] != 0;
}

// Grid-mask bits of a run of `n` (<= 64) consecutive local key rows [k0, k0+n) for one
// query position: bit i set = key k0+i hidden.  One table lookup when the run stays in
// one key cell (the common case), per key otherwise.
__device__ __forceinline__ uint64_t grid_key_bits(const burst_hop& h, int64_t qp, int64_t k0, int n) {
  const uint32_t row = grid_qc(h, qp) * (uint32_t)h.grid_nkb;
  const int64_t kp0 = pos_of(h.k_map, k0), kp1 = pos_of(h.k_map, k0 + n - 1);
  const uint32_t c0 = grid_kc(h, kp0);
  if (kp1 - kp0 == n - 1 && c0 == grid_kc(h, kp1))
    return h.grid_skip[row + c0] ? (n == 64 ? ~0ull : ((1ull << n) - 1)) : 0ull;
  uint64_t bits = 0;
  for (int i = 0; i < n; ++i)
    if (h.grid_skip[row + grid_kc(h, pos_of(h.k_map, k0 + i))]) bits |= 1ull << i;
  return bits;
}

// Same for a run of `n` (<= 64) consecutive local query rows against one key position.
__device__ __forceinline__ uint64_t grid_query_bits(const burst_hop& h, int64_t q0, int n, int64_t kp) {
  const uint32_t col = grid_kc(h, kp), nkb = (uint32_t)h.grid_nkb;
  const int64_t qp0 = pos_of(h.q_map, q0), qp1 = pos_of(h.q_map, q0 + n - 1);
  const uint32_t c0 = grid_qc(h, qp0);
  if (qp1 - qp0 == n - 1 && c0 == grid_qc(h, qp1))
    return h.grid_skip[c0 * nkb + col] ? (n == 64 ? ~0ull : ((1ull << n) - 1)) : 0ull;
  uint64_t bits = 0;
  for (int i = 0; i < n; ++i)
    if (h.grid_skip[grid_qc(h, pos_of(h.q_map, q0 + i)) * nkb + col]) bits |= 1ull << i;
  return bits;
}

// Does the rectangle of local query rows [q0, q0+nq) x local key rows [k0, k0+nk)
// contain a (query, key) pair outside the skipped grid cells?  Cell-granular (a
// partially skipped tile counts as live; its elements are masked separately).
// Every role of a kernel evaluates it identically, so tiles it rejects are skipped
// by all of them (the SKIP decision of BlockMask.decision, masking.py:79-106).
__device__ __forceinline__ void grid_cells_of(const burst_posmap& m, int64_t r0, int64_t n,
                                              uint32_t cell, uint32_t ncells, uint32_t (&lo)[2],
                                              uint32_t (&hi)[2]) {
  // at most two contiguous position segments: rows before / after seg_len
  lo[0] = lo[1] = 1;
  hi[0] = hi[1] = 0;                    // empty unless set below
  const int64_t a0 = r0, a1 = (r0 + n < m.seg_len ? r0 + n : m.seg_len);
  if (a1 > a0) {
    lo[0] = (uint32_t)(m.pos0 + a0) / cell;
    hi[0] = (uint32_t)(m.pos0 + a1 - 1) / cell;
  }
  const int64_t b0 = (r0 > m.seg_len ? r0 : m.seg_len), b1 = r0 + n;
  if (b1 > b0) {
    lo[1] = (uint32_t)(m.pos1 + b0 - m.seg_len) / cell;
    hi[1] = (uint32_t)(m.pos1 + b1 - 1 - m.seg_len) / cell;
  }
  for (int s = 0; s < 2; ++s) {             // padding rows read the last cell (grid_qc)
    if (lo[s] >= ncells && lo[s] <= hi[s]) lo[s] = ncells - 1;
    if (hi[s] >= ncells) hi[s] = ncells - 1;
  }
}
__device__ __forceinline__ bool grid_rect_live(const burst_hop& h, int64_t q0, int64_t nq,
                                               int64_t k0, int64_t nk) {
  if (!h.grid_skip || nq <= 0 || nk <= 0) return true;
  uint32_t ql[2], qh[2], kl[2], kh[2];
  const uint32_t nkb = (uint32_t)h.grid_nkb;
  grid_cells_of(h.q_map, q0, nq, (uint32_t)h.grid_qcell, (uint32_t)h.grid_nqb, ql, qh);
  grid_cells_of(h.k_map, k0, nk, (uint32_t)h.grid_kcell, nkb, kl, kh);
  for (int a = 0; a < 2; ++a)
    for (uint32_t qc = ql[a]; qc <= qh[a]; ++qc)
      for (int b = 0; b < 2; ++b)
        for (uint32_t kc = kl[b]; kc <= kh[b]; ++kc)
          if (!h.grid_skip[qc * nkb + kc]) return true;
  return false;
}

// ... and is every pair of the rectangle outside the skipped cells (no element masking
// needed inside it)?
__device__ __forceinline__ bool grid_rect_full(const burst_hop& h, int64_t q0, int64_t nq,
                                               int64_t k0, int64_t nk) {
  if (!h.grid_skip || nq <= 0 || nk <= 0) return true;
  uint32_t ql[2], qh[2], kl[2], kh[2];
  const uint32_t nkb = (uint32_t)h.grid_nkb;
  grid_cells_of(h.q_map, q0, nq, (uint32_t)h.grid_qcell, (uint32_t)h.grid_nqb, ql, qh);
  grid_cells_of(h.k_map, k0, nk, (uint32_t)h.grid_kcell, nkb, kl, kh);
  for (int a = 0; a < 2; ++a)
    for (uint32_t qc = ql[a]; qc <= qh[a]; ++qc)
      for (int b = 0; b < 2; ++b)
        for (uint32_t kc = kl[b]; kc <= kh[b]; ++kc)
          if (h.grid_skip[qc * nkb + kc]) return false;
  return true;
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
