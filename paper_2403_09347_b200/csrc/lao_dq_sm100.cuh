// Deterministic dQ of the LAO backward on sm_100a (used when burst_hop.dq_order is set).
//
// The fused backward (lao_bwd4) walks key-stationary and reduces each step's fp32 dQ
// partial into a shared accumulator, so the summation order depends on timing.  In
// deterministic mode lao_bwd4 computes dK/dV only, and this kernel computes dQ
// query-stationary: each CTA owns 128 query rows, recomputes S = Q K^T and
// dP = dO V^T for every visible key tile, forms dS = P o (dP - D) with
// P = exp2(S * scale*log2e - lse*log2e) (local_attn.py:298-307), accumulates
// dQ += dS K in TMEM in key-tile order and adds it to dq_acc once at the end -- one
// writer per dQ row, so the result is bit-reproducible (pkg/tests/test_sim.py:280-295).
// Costs two extra MMAs per tile (S, dP) against the ordered reductions it replaces.
//
//   warps 0-7  dS for keys [0,64) (warps 0-3) / [64,128) (warps 4-7) of each tile,
//              thread = query row = TMEM lane; then the dQ epilogue (column halves)
//   warp  8    TMA producer (+ TMEM allocator)
//   warp  9    tcgen05.mma issuer (one elected lane)
// TMEM (512 cols): S0 [0,128) S1 [128,256) (dS, bf16, over the first 32 columns of
// each key half of S_b once read) | dP [256,384) | dQ [384,384+D).
#pragma once
#include <cuda.h>
#include "common.cuh"
#include "ptx.cuh"

namespace burst {
namespace bdq {

constexpr int BM = 128;        // query rows per CTA
constexpr int BN = 128;        // keys per tile
constexpr int kThreads = 384;  // 3 warpgroups (warps 10-11 idle) for setmaxnreg

template <int D>
struct Cfg {
  static constexpr int kBoxBytes = 128 * 64 * 2;
  static constexpr int kBoxes = D / 64;
  static constexpr int kTileBytes = kBoxBytes * kBoxes;
  // K_j and V_j occupy one slot each (items 2j, 2j+1 of the load stream): V_j is free
  // after dP_j, K_j after dQ_j, so the loads run up to two tiles ahead of the MMAs
  static constexpr int kSlots = (D == 128) ? 5 : 8;
  static constexpr int kLiveWords = 256;     // live-key-tile bitmap (grid masks): 8192 tiles
  static constexpr int kSmemBytes = 1024 + 2 * kTileBytes + kSlots * kTileBytes + 256 +
                                    4 * kLiveWords;
};

struct Params {
  CUtensorMap tm_q, tm_do, tm_k, tm_v;
  const float* stats;   // [2][B*H][NTq*128]: lse*log2e, D
  float* dq_acc;        // TL over n_q
  burst_hop hop;
  float scale_log2, scale;
};

template <int D, bool kGrid>
__global__ void __launch_bounds__(kThreads, 1) lao_dq_kernel(const __grid_constant__ Params p) {
  using C = Cfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem;
  {
    const uint32_t s = ptx::smem_u32(smem_raw);
    smem = smem_raw + ((1024u - (s & 1023u)) & 1023u);
  }
  uint8_t* sQ = smem;
  uint8_t* sdO = sQ + C::kTileBytes;
  uint8_t* sKV = sdO + C::kTileBytes;   // kSlots slots: K_j, V_j alternate
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + C::kSlots * C::kTileBytes);
  uint64_t* q_full = bars;                       // Q and dO landed
  uint64_t* kv_full = bars + 1;                  // [kSlots]
  uint64_t* kv_empty = kv_full + C::kSlots;      // [kSlots]
  uint64_t* s_full = kv_empty + C::kSlots;       // [2] S_b computed
  uint64_t* s_free = s_full + 2;                 // [2] dQ MMA done reading dS in S_b
  uint64_t* ds_full = s_free + 2;                // [2] dS in S_b (256 arrivals)
  uint64_t* dp_full = ds_full + 2;
  uint64_t* dp_free = dp_full + 1;               // dP read into registers (256 arrivals)
  uint64_t* dq_done = dp_free + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(dq_done + 1);
  uint32_t* live_bits = reinterpret_cast<uint32_t*>(bars + 32);

  const burst_hop& hp = p.hop;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.z, h = blockIdx.y;
  const int64_t bh = (int64_t)b * hp.heads + h;
  const int64_t q_end = hp.q_begin + hp.q_len;
  const int64_t row0 = hp.q_begin + (int64_t)blockIdx.x * BM;
  const int64_t qrows = (row0 + BM < q_end ? row0 + BM : q_end) - row0;
  const int64_t NTq = ceil_div(hp.n_q, 128);

  // Key span of this query tile: causal => a prefix of the hop's keys (monotone maps).
  int64_t kspan = hp.k_len;
  if (hp.causal) {
    const int64_t cnt = count_le(hp.k_map, hp.n_k, pos_of(hp.q_map, row0 + qrows - 1)) - hp.k_begin;
    kspan = cnt < kspan ? cnt : kspan;
    if (kspan < 0) kspan = 0;
  }
  const int nkv = (int)ceil_div(kspan, BN);
  auto live = [&](int j) -> bool {
    if (!kGrid) return true;
    if (j >= nkv) return false;
    const int64_t kr = kspan - (int64_t)j * BN;
    return grid_rect_live(hp, row0, qrows, hp.k_begin + (int64_t)j * BN, kr < BN ? kr : BN);
  };
  const bool use_bits = kGrid && nkv <= C::kLiveWords * 32;
  if (use_bits) {
    for (int w = threadIdx.x; w < ((nkv + 31) >> 5); w += kThreads) live_bits[w] = 0u;
    __syncthreads();
    for (int j = threadIdx.x; j < nkv; j += kThreads)
      if (live(j)) atomicOr(live_bits + (j >> 5), 1u << (j & 31));
    __syncthreads();
  }
  auto next_live = [&](int j) -> int {
    if (!kGrid) return j;
    if (use_bits) {
      if (j >= nkv) return nkv;
      int w = j >> 5;
      uint32_t m = live_bits[w] & (~0u << (j & 31));
      const int nw = (nkv + 31) >> 5;
      while (m == 0u) {
        if (++w >= nw) return nkv;
        m = live_bits[w];
      }
      const int r = (w << 5) + __ffs(m) - 1;
      return r < nkv ? r : nkv;
    }
    while (j < nkv && !live(j)) ++j;
    return j;
  };
  const int first = next_live(0);
  const bool any = first < nkv;

  if (warp == 8) {
    if (lane == 0) {
      ptx::mbar_init(q_full, 1);
      for (int s = 0; s < C::kSlots; ++s) {
        ptx::mbar_init(kv_full + s, 1);
        ptx::mbar_init(kv_empty + s, 1);
      }
      for (int t = 0; t < 2; ++t) {
        ptx::mbar_init(s_full + t, 1);
        ptx::mbar_init(s_free + t, 1);
        ptx::mbar_init(ds_full + t, 2 * BM);
      }
      ptx::mbar_init(dp_full, 1);
      ptx::mbar_init(dp_free, 2 * BM);
      ptx::mbar_init(dq_done, 1);
      ptx::fence_mbar_init();
      ptx::tma_prefetch_desc(&p.tm_q);
      ptx::tma_prefetch_desc(&p.tm_do);
      ptx::tma_prefetch_desc(&p.tm_k);
      ptx::tma_prefetch_desc(&p.tm_v);
    }
    __syncwarp();
    ptx::tmem_alloc(tmem_holder, 512);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = *tmem_holder;
  constexpr uint32_t kDP = 256, kDQ = 384;

  if (warp >= 8) {
    ptx::regs_dec<88>();
    if (warp == 8) {
      // ---------------------------------------------------------- TMA producer
      if (lane == 0 && any) {
        ptx::mbar_expect_tx(q_full, 2 * C::kTileBytes);
        for (int x = 0; x < C::kBoxes; ++x) {
          ptx::tma_load_4d(sQ + x * C::kBoxBytes, &p.tm_q, q_full, x * 64, h, (int)row0, b);
          ptx::tma_load_4d(sdO + x * C::kBoxBytes, &p.tm_do, q_full, x * 64, h, (int)row0, b);
        }
        int it = 0;
        for (int u = first; u < nkv; u = next_live(u + 1)) {
          const int krow = (int)(hp.k_begin + (int64_t)u * BN);
          for (int kv = 0; kv < 2; ++kv, ++it) {
            const int s = it % C::kSlots;
            const uint32_t use = it / C::kSlots;
            ptx::mbar_wait(kv_empty + s, (use & 1) ^ 1);
            ptx::mbar_expect_tx(kv_full + s, C::kTileBytes);
            for (int x = 0; x < C::kBoxes; ++x)
              ptx::tma_load_4d(sKV + s * C::kTileBytes + x * C::kBoxBytes, kv == 0 ? &p.tm_k : &p.tm_v,
                               kv_full + s, x * 64, h, krow, b);
          }
        }
      }
    } else if (warp == 9) {
      // ---------------------------------------------------------- MMA issuer
      // Per live key tile jj (S double-buffered): S_{jj+1} | dP_{jj+1} once dP_jj is in
      // registers | dQ += dS_jj K_jj once dS_jj is in TMEM.
      if (any) {
        constexpr uint32_t id_qk = ptx::make_idesc_bf16(BM, BN, 0, 0);   // S, dP (K-major)
        constexpr uint32_t id_dq = ptx::make_idesc_bf16(BM, D, 0, 1);    // A TMEM, B MN-major
        const uint64_t dQk = ptx::make_sdesc(ptx::smem_u32(sQ), 0, 1024);
        const uint64_t dOk = ptx::make_sdesc(ptx::smem_u32(sdO), 0, 1024);
        const uint64_t dKVk = ptx::make_sdesc(ptx::smem_u32(sKV), 0, 1024);
        const uint64_t dKVm = ptx::make_sdesc(ptx::smem_u32(sKV), C::kBoxBytes, 1024);
        constexpr uint64_t kTile = (uint64_t)(C::kTileBytes >> 4);
        auto kmaj = [](int kk) -> uint64_t { return (uint64_t)(((kk >> 2) * C::kBoxBytes + (kk & 3) * 32) >> 4); };
        // item it of the load stream (K_j = 2j, V_j = 2j + 1): its slot and fill parity
        auto slot = [](int it) -> int { return it % C::kSlots; };
        auto wait_item = [&](int it) { ptx::mbar_wait(kv_full + slot(it), (it / C::kSlots) & 1); };
        auto s_mma = [&](int buf, int jj) {   // S_buf = Q K_jj^T
          if (ptx::elect_one()) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk)
              ptx::mma_ss(tbase + buf * 128, dQk + kmaj(kk), dKVk + slot(2 * jj) * kTile + kmaj(kk), id_qk,
                          kk > 0);
            ptx::mma_commit(s_full + buf);
          }
          __syncwarp();
        };
        auto dp_mma = [&](int jj) {   // dP = dO V_jj^T; V_jj's last reader
          if (ptx::elect_one()) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk)
              ptx::mma_ss(tbase + kDP, dOk + kmaj(kk), dKVk + slot(2 * jj + 1) * kTile + kmaj(kk), id_qk,
                          kk > 0);
            ptx::mma_commit(dp_full);
            ptx::mma_commit(kv_empty + slot(2 * jj + 1));
          }
          __syncwarp();
        };
        auto dq_mma = [&](int buf, int jj) {   // dQ += dS K_jj (A = dS from TMEM); K_jj's last reader
          if (ptx::elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BN / 16; ++kk)
              ptx::mma_ts(tbase + kDQ, tbase + buf * 128 + (kk < 4 ? kk * 8 : 32 + kk * 8),
                          dKVm + slot(2 * jj) * kTile + (uint64_t)(kk * 2048 >> 4), id_dq,
                          (jj > 0 || kk > 0) ? 1u : 0u);
            ptx::mma_commit(s_free + buf);
            ptx::mma_commit(kv_empty + slot(2 * jj));
          }
          __syncwarp();
        };
        ptx::mbar_wait(q_full, 0);
        wait_item(0);
        ptx::tc_fence_after();
        s_mma(0, 0);
        wait_item(1);
        ptx::tc_fence_after();
        dp_mma(0);
        for (int u = first, jj = 0; u < nkv; ++jj) {
          const int un = next_live(u + 1);
          const int buf = jj & 1;
          if (un < nkv) {
            wait_item(2 * jj + 2);
            if (jj >= 1) ptx::mbar_wait(s_free + (buf ^ 1), ((jj - 1) >> 1) & 1);
            ptx::tc_fence_after();
            s_mma(buf ^ 1, jj + 1);
            ptx::mbar_wait(dp_free, jj & 1);
            wait_item(2 * jj + 3);
            ptx::tc_fence_after();
            dp_mma(jj + 1);
          }
          ptx::mbar_wait(ds_full + buf, (jj >> 1) & 1);
          ptx::tc_fence_after();
          dq_mma(buf, jj);
          u = un;
        }
        if (ptx::elect_one()) ptx::mma_commit(dq_done);
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ dS warpgroups
    ptx::regs_inc<208>();
    const int hk = warp >> 2;                 // key half of every tile
    const int t = threadIdx.x & 127;          // query row within the tile = TMEM lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int64_t row = row0 + t;
    const bool valid = row < q_end && row < hp.n_q;
    const int64_t srow = valid ? row : row0;
    const float lse2 = p.stats[bh * NTq * 128 + srow];
    const float Dv = p.stats[((int64_t)hp.batch * hp.heads + bh) * NTq * 128 + srow];
    const int64_t qpos = pos_of(hp.q_map, srow);
    int64_t lim = hp.k_len;   // keys visible to this row, relative to k_begin
    if (hp.causal) {
      const int64_t cnt = count_le(hp.k_map, hp.n_k, qpos) - hp.k_begin;
      lim = cnt < lim ? cnt : lim;
    }
    if (!valid) lim = 0;
    const float c2 = p.scale_log2;
    for (int u = first, jj = 0; u < nkv; u = next_live(u + 1), ++jj) {
      const int buf = jj & 1;
      const int64_t k0 = (int64_t)u * BN + 64 * hk;   // first key of this half, rel. k_begin
      const int64_t nv64 = lim - k0;
      const int nv = nv64 > 64 ? 64 : (nv64 < 0 ? 0 : (int)nv64);
      uint64_t gk = 0;   // block-sparse grid: hidden key columns of this row
      if (kGrid && hp.grid_skip && nv > 0) gk = grid_key_bits(hp, qpos, hp.k_begin + k0, nv);
      ptx::mbar_wait(s_full + buf, (jj >> 1) & 1);
      ptx::tc_fence_after();
      // P from S while dP_jj is still being computed, then dS once dP_jj is in registers
      const bool full = __all_sync(0xffffffffu, nv == 64 && gk == 0);
      float pr[64];
      {
        uint32_t r[64];
        ptx::tmem_ld32(tbase + lane_off + buf * 128 + 64 * hk, *reinterpret_cast<uint32_t(*)[32]>(r));
        ptx::tmem_ld32(tbase + lane_off + buf * 128 + 64 * hk + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
        ptx::tmem_wait_ld();
        ptx::reg_fence(r);
#pragma unroll
        for (int c = 0; c < 64; c += 2) {
          const float2 x = ptx::ffma2(make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])),
                                      make_float2(c2, c2), make_float2(-lse2, -lse2));
          pr[c] = ptx::ex2(x.x);
          pr[c + 1] = ptx::ex2(x.y);
        }
      }
      if (!full) {
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (c >= nv || ((gk >> c) & 1)) pr[c] = 0.f;
      }
      ptx::mbar_wait(dp_full, jj & 1);
      ptx::tc_fence_after();
      uint32_t d[64];
      ptx::tmem_ld32(tbase + lane_off + kDP + 64 * hk, *reinterpret_cast<uint32_t(*)[32]>(d));
      ptx::tmem_ld32(tbase + lane_off + kDP + 64 * hk + 32, *reinterpret_cast<uint32_t(*)[32]>(d + 32));
      ptx::tmem_wait_ld();
      ptx::reg_fence(d);
      ptx::tc_fence_before();
      ptx::mbar_arrive(dp_free);   // dP_{jj+1} may overwrite the dP columns
      uint32_t pk[32];
#pragma unroll
      for (int c = 0; c < 64; c += 2) {
        // dS = P * (dP - D)
        const float2 ds = ptx::fmul2(make_float2(pr[c], pr[c + 1]),
                                     ptx::fadd2(make_float2(__uint_as_float(d[c]), __uint_as_float(d[c + 1])),
                                                make_float2(-Dv, -Dv)));
        pk[c >> 1] = ptx::pack_bf16(ds.x, ds.y);
      }
      ptx::tmem_st32(tbase + lane_off + buf * 128 + 64 * hk, pk);
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive(ds_full + buf);
    }
    // -------------------------------------------------------- dQ epilogue
    if (any) {
      ptx::mbar_wait(dq_done, 0);
      ptx::tc_fence_after();
#pragma unroll 1
      for (int cc = hk * (D / 64); cc < (hk + 1) * (D / 64); ++cc) {
        uint32_t r[32];
        ptx::tmem_ld32(tbase + lane_off + kDQ + cc * 32, r);
        ptx::tmem_wait_ld();
        ptx::reg_fence(r);
        if (!valid) continue;
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float4* a = reinterpret_cast<float4*>(p.dq_acc + tl_index(bh, row, cc * 32 + j, D, NTq));
          const float4 o = *a;
          *a = make_float4(o.x + __uint_as_float(r[j]) * p.scale, o.y + __uint_as_float(r[j + 1]) * p.scale,
                           o.z + __uint_as_float(r[j + 2]) * p.scale, o.w + __uint_as_float(r[j + 3]) * p.scale);
        }
      }
    }
  }

  __syncwarp();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tbase, 512);
  }
}

}  // namespace bdq
}  // namespace burst
