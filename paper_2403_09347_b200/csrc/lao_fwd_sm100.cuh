// LAO forward on sm_100a: TMA -> SMEM (128B swizzle) -> tcgen05.mma -> TMEM,
// online softmax in registers, P written back to TMEM and consumed by a
// TMEM-operand MMA, GAO merge with the running (O_acc, m, l) state fused into
// the epilogue.
//
// Reference semantics: one call = ring.forward_step (ring.py:158-181) for every
// (batch, head) slice: local_forward_tiled (local_attn.py:207-248) over the
// hop's rectangle followed by PartialAttn.merge into the device state
// (local_attn.py:101-120), and on the last hop PartialAttn.finalize
// (local_attn.py:127-135).  Scores use S * scale * log2(e) with exp2; the state
// keeps m in log2 units; lse is converted back to natural log.
//
// CTA = 2 query tiles of 128 rows sharing every K/V tile (halves K/V SMEM and
// L2 traffic per FLOP and lets one tile's softmax overlap the other's MMAs).
//   warps 0-3  softmax/epilogue for query tile 0 (thread = row = TMEM lane)
//   warps 4-7  softmax/epilogue for query tile 1
//   warp  8    TMA producer (+ TMEM allocator)
//   warp  9    tcgen05.mma issuer (one elected lane)
// TMEM (512 cols): S0 [0,128) S1 [128,256) O0 [256,256+D) O1 [256+D,256+2D);
// P_t (bf16, 64 cols) aliases the first half of S_t.
#pragma once
#include <cuda.h>
#include <type_traits>
#include "common.cuh"
#include "ptx.cuh"

namespace burst {
namespace fwd {

constexpr int BM = 128;       // query rows per tile
constexpr int BN = 128;       // keys per tile
constexpr int kThreads = 384;   // 3 warpgroups (warps 10-11 idle) for setmaxnreg
#ifndef BURST_FWD_PSPLIT   // key chunks of P handed to the O += P V MMAs one at a time
#define BURST_FWD_PSPLIT 2
#endif
constexpr int kPS = BURST_FWD_PSPLIT;        // 1, 2 or 4
constexpr float kRescaleThreshold = 8.0f;  // log2 units: lazy rescale (values <= 2^8)

template <int D>
struct Cfg {
  static constexpr int kBoxBytes = 128 * 64 * 2;      // one TMA box: 128 rows x 64 bf16
  static constexpr int kBoxes = D / 64;
  static constexpr int kTileBytes = kBoxBytes * kBoxes;
  static constexpr int kStages = (D == 128) ? 4 : 6;
  static constexpr int kLiveWords = 256;   // live-KV-tile bitmap (grid masks): 8192 tiles
  static constexpr int kSmemBytes = 1024 + 2 * kTileBytes + kStages * kTileBytes + 256 + 8 * kLiveWords;
};

struct Params {
  CUtensorMap tm_q, tm_k, tm_v;
  float* o_acc;
  float* m_run;
  float* l_run;
  void* o_out;
  float* lse_out;
  int* flags;
  burst_hop hop;
  float scale_log2;
  int first_hop, finalize;
  long long* trace;   // BURST_TRACE builds only: per-iteration clock64 timeline
};

#ifdef BURST_TRACE
#define FTRACE(ev, i)                                                                        \
  do {                                                                                       \
    if (p.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (i) < 64)        \
      p.trace[(ev) * 64 + (i)] = clock64();                                                  \
  } while (0)
#else
#define FTRACE(ev, i)
#endif

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  uintptr_t a = reinterpret_cast<uintptr_t>(p);
  uint32_t s = ptx::smem_u32(p);
  uint32_t pad = (1024u - (s & 1023u)) & 1023u;
  return reinterpret_cast<uint8_t*>(a + pad);
}

// kGrid: the general instantiation -- the hop carries a block-sparse grid mask (tile
// skipping + element masks) and/or a key-tile visiting order (burst_hop.key_order,
// local_forward_tiled's key_tile_order, local_attn.py:212-225); the dense instantiation
// keeps its loops free of that bookkeeping.  Roles walk "visit" indices u; tile j =
// key_order[u] (or u).
// kPair: launched as 2-CTA clusters over adjacent query blocks that walk the SAME key
// tiles; each CTA TMA-loads one 64-column box of every K and V tile with
// .multicast::cluster into both (half the L2 reads of K/V); a stage is refilled once
// both CTAs released it (2-count empty barriers fed by multicast tcgen05.commit).
template <int D, bool kGrid, bool kPair = false>
__global__ void __launch_bounds__(kThreads, 1) lao_fwd_kernel(const __grid_constant__ Params p) {
  using C = Cfg<D>;
  static_assert(!kPair || D == 128, "the paired forward splits K/V tiles by 64-column box");
  // FMA-pipe exp2 share (profiles/r01_poly_exp2.txt): 5/16 measured best for dense hops,
  // 3/8 for the grid-masked instantiation (c3_sparse: 122.5 vs 126.3 ms per launch)
  constexpr int kPolyMod = kGrid ? 8 : BURST_POLY_MOD;
  constexpr int kPolyCnt = kGrid ? 3 : BURST_POLY_CNT;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sQ = smem;                          // 2 tiles
  uint8_t* sKV = smem + 2 * C::kTileBytes;     // kStages slots (K_j, V_j alternate)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + C::kStages * C::kTileBytes);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + C::kStages;
  uint64_t* s_full = kv_empty + C::kStages;   // [2]
  uint64_t* p_full = s_full + 2;              // [2 tiles][kPS key chunks]
  uint64_t* o_full = p_full + 2 * kPS;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(o_full + 1);

  const burst_hop& hp = p.hop;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.z, h = blockIdx.y;
  const int64_t q_end = hp.q_begin + hp.q_len;
  // causal: later query rows see more keys, so launch them first (longest-first
  // order shortens the tail wave of the grid)
  const int64_t xb = hp.causal ? (int64_t)(gridDim.x - 1 - blockIdx.x) : (int64_t)blockIdx.x;
  const int64_t row0 = hp.q_begin + xb * (2 * BM);
  // the query rows whose key walk this CTA follows: its own 256, or its pair's 512
  const uint32_t crank = kPair ? ptx::cluster_rank() : 0u;
  const int64_t xb_peer = hp.causal ? (int64_t)(gridDim.x - 1 - (blockIdx.x ^ 1u)) : (int64_t)(blockIdx.x ^ 1u);
  const int64_t wrow0 = kPair ? hp.q_begin + (xb < xb_peer ? xb : xb_peer) * (2 * BM) : row0;
  const int64_t wrow1 = wrow0 + (kPair ? 4 : 2) * BM;   // exclusive

  // Key span this CTA needs: causal => a prefix of the hop's keys (monotone maps).
  int64_t kspan = hp.k_len;
  if (hp.causal) {
    int64_t last = (wrow1 < q_end ? wrow1 : q_end) - 1;
    int64_t cnt = count_le(hp.k_map, hp.n_k, pos_of(hp.q_map, last)) - hp.k_begin;
    kspan = cnt < kspan ? cnt : kspan;
    if (kspan < 0) kspan = 0;
  }
  const int nkv = (int)ceil_div(kspan, BN);
  // Visiting order: with key_order the walk covers every key tile of the hop and the
  // ones past the causal span are skipped like grid-dead tiles.
  const int32_t* korder = kGrid ? hp.key_order : nullptr;
  const int nu = korder ? (int)ceil_div(hp.k_len, BN) : nkv;
  auto tile_at = [&](int u) -> int { return korder ? __ldg(korder + u) : u; };
  // Block-sparse grid: KV tiles whose every (query, key) pair lies in skipped cells
  // are skipped by every role (each evaluates the same predicate).
  const int64_t qrows = (row0 + 2 * BM < q_end ? row0 + 2 * BM : q_end) - row0;
  const int64_t wrows = (wrow1 < q_end ? wrow1 : q_end) - wrow0;
  auto live = [&](int j) -> bool {   // (kPair: live for either CTA of the pair)
    if (!kGrid) return true;
    if (j >= nkv) return false;
    const int64_t kr = kspan - (int64_t)j * BN;
    return grid_rect_live(hp, wrow0, wrows, hp.k_begin + (int64_t)j * BN, kr < BN ? kr : BN);
  };
  // The predicate is evaluated once per tile by the whole CTA into a SMEM bitmap (up to
  // kLiveWords * 32 tiles); every role then finds the next live tile with __ffs.  A
  // second bitmap marks tiles lying wholly inside visible cells: the softmax skips the
  // per-row grid bits there.
  uint32_t* live_bits = reinterpret_cast<uint32_t*>(bars + 32);
  uint32_t* full_bits = live_bits + C::kLiveWords;
  const bool use_bits = kGrid && !korder && nkv <= C::kLiveWords * 32;
  if (use_bits) {
    const int nw = (nkv + 31) >> 5;
    for (int w = threadIdx.x; w < nw; w += kThreads) live_bits[w] = full_bits[w] = 0u;
    __syncthreads();
    for (int j = threadIdx.x; j < nkv; j += kThreads) {
      if (live(j)) atomicOr(live_bits + (j >> 5), 1u << (j & 31));
      const int64_t kr = kspan - (int64_t)j * BN;
      if (grid_rect_full(hp, row0, qrows, hp.k_begin + (int64_t)j * BN, kr < BN ? kr : BN))
        atomicOr(full_bits + (j >> 5), 1u << (j & 31));
    }
    __syncthreads();
  }
  auto next_live = [&](int j) -> int {   // next visit index u >= j of a live tile
    if (!kGrid) return j;
    if (korder) {
      while (j < nu && !live(tile_at(j))) ++j;
      return j;
    }
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
  const bool any = first < nu;

  if (warp == 8) {
    if (lane == 0) {
      ptx::mbar_init(q_full, 1);
      for (int s = 0; s < C::kStages; ++s) {
        ptx::mbar_init(kv_full + s, 1);
        ptx::mbar_init(kv_empty + s, kPair ? 2 : 1);
      }
      for (int t = 0; t < 2; ++t) {
        ptx::mbar_init(s_full + t, 1);
        for (int c = 0; c < kPS; ++c) ptx::mbar_init(p_full + kPS * t + c, BM);
      }
      ptx::mbar_init(o_full, 1);
      ptx::fence_mbar_init();
      ptx::tma_prefetch_desc(&p.tm_q);
      ptx::tma_prefetch_desc(&p.tm_k);
      ptx::tma_prefetch_desc(&p.tm_v);
    }
    __syncwarp();
    ptx::tmem_alloc(tmem_holder, 512);
  }
  ptx::tc_fence_before();
  if (kPair)
    ptx::cluster_sync();   // both CTAs' barriers exist before either multicasts into them
  else
    __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = *tmem_holder;
  if (warp >= 8) {
   ptx::regs_dec<88>();
   if (warp == 8) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && any) {
      ptx::mbar_expect_tx(q_full, 2 * C::kTileBytes);
      for (int t = 0; t < 2; ++t)
        for (int x = 0; x < C::kBoxes; ++x)
          ptx::tma_load_4d(sQ + t * C::kTileBytes + x * C::kBoxBytes, &p.tm_q, q_full, x * 64, h,
                           (int)(row0 + t * BM), b);
      int it = 0;
      for (int u = first; u < nu; u = next_live(u + 1)) {
        const int krow = (int)(hp.k_begin + (int64_t)tile_at(u) * BN);
        for (int kv = 0; kv < 2; ++kv, ++it) {
          const int s = it % C::kStages;
          const uint32_t use = it / C::kStages;
          ptx::mbar_wait(kv_empty + s, (use & 1) ^ 1);
          ptx::mbar_expect_tx(kv_full + s, C::kTileBytes);
          const CUtensorMap* tm = kv == 0 ? &p.tm_k : &p.tm_v;
          if (kPair)
            ptx::tma_load_4d_mc(sKV + s * C::kTileBytes + crank * C::kBoxBytes, tm, kv_full + s,
                                (int)crank * 64, h, krow, b, 3);
          else
            for (int x = 0; x < C::kBoxes; ++x)
              ptx::tma_load_4d(sKV + s * C::kTileBytes + x * C::kBoxBytes, tm, kv_full + s, x * 64,
                               h, krow, b);
        }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    // Whole warp runs the loop (uniform control flow keeps descriptors in uniform
    // registers); one elected lane issues each MMA group and its commits.
    if (any) {
      constexpr uint32_t idesc_qk = ptx::make_idesc_bf16(BM, BN, 0, 0);
      constexpr uint32_t idesc_pv = ptx::make_idesc_bf16(BM, D, 0, 1);
      const uint64_t dQk = ptx::make_sdesc(ptx::smem_u32(sQ), 0, 1024);
      const uint64_t dKVk = ptx::make_sdesc(ptx::smem_u32(sKV), 0, 1024);            // K (K-major)
      const uint64_t dKVm = ptx::make_sdesc(ptx::smem_u32(sKV), C::kBoxBytes, 1024); // V (MN-major)
      constexpr uint64_t kTile = (uint64_t)(C::kTileBytes >> 4);
      auto qk = [&](int t, int slot) {
        if (ptx::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t off = (uint64_t)(((kk >> 2) * C::kBoxBytes + (kk & 3) * 32) >> 4);
            ptx::mma_ss(tbase + t * 128, dQk + t * kTile + off, dKVk + slot * kTile + off, idesc_qk,
                        kk > 0);
          }
          ptx::mma_commit(s_full + t);
        }
        __syncwarp();
      };
      // O_t += P_t V in kPS key chunks: a chunk's MMAs start as soon as the softmax has
      // stored its P, overlapping the exp2 of the following keys
      auto pv = [&](int t, int slot, bool acc, int chunk) {
        if (ptx::elect_one()) {
#pragma unroll
          for (int k4 = 0; k4 < BN / 16 / kPS; ++k4) {
            const int kk = chunk * (BN / 16 / kPS) + k4;
            ptx::mma_ts(tbase + 256 + t * D, tbase + t * 128 + kk * 8,
                        dKVm + slot * kTile + (uint64_t)(kk * 2048 >> 4), idesc_pv,
                        (acc || kk > 0) ? 1u : 0u);
          }
        }
        __syncwarp();
      };
      auto commit = [&](uint64_t* b) {
        if (ptx::elect_one()) ptx::mma_commit(b);
        __syncwarp();
      };
      auto release = [&](uint64_t* b) {   // a K/V stage: this CTA is done with it (in both)
        if (ptx::elect_one()) {
          if (kPair)
            ptx::mma_commit_mc(b, 3);
          else
            ptx::mma_commit(b);
        }
        __syncwarp();
      };
      ptx::mbar_wait(q_full, 0);
      ptx::mbar_wait(kv_full + 0, 0);
      ptx::tc_fence_after();
      qk(0, 0);
      qk(1, 0);
      release(kv_empty + 0);
      // jj = index among the live KV tiles (stage / parity counter); j = tile index
      for (int j = first, jj = 0; j < nu; ++jj) {
        const int jn = next_live(j + 1);
        const int itv = 2 * jj + 1, sv = itv % C::kStages;
        const int itk = 2 * jj + 2, sk = itk % C::kStages;
        const bool more = jn < nu;
        ptx::mbar_wait(kv_full + sv, (itv / C::kStages) & 1); FTRACE(0, jj);
        for (int c = 0; c < kPS; ++c) {
          ptx::mbar_wait(p_full + c, jj & 1); if (c == 0) FTRACE(1, jj);
          ptx::tc_fence_after();
          pv(0, sv, jj > 0, c);
        }
        if (more) {
          ptx::mbar_wait(kv_full + sk, (itk / C::kStages) & 1);
          ptx::tc_fence_after();
          qk(0, sk);
        }
        for (int c = 0; c < kPS; ++c) {
          ptx::mbar_wait(p_full + kPS + c, jj & 1); if (c == 0) FTRACE(2, jj);
          ptx::tc_fence_after();
          pv(1, sv, jj > 0, c);
        }
        release(kv_empty + sv);
        if (more) {
          qk(1, sk);
          release(kv_empty + sk);
        }
        j = jn;
      }
      commit(o_full);
    }
   }
  } else {
    // ------------------------------------------------------------ softmax WGs
    ptx::regs_inc<208>();
    const int g = warp >> 2;                 // query tile 0/1
    const int t = threadIdx.x & 127;         // row within the tile = TMEM lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tS = tbase + lane_off + g * 128;
    const uint32_t tO = tbase + lane_off + 256 + g * D;
    const int64_t row = row0 + g * BM + t;
    const bool valid = row < q_end && row < hp.n_q;
    // keys visible to this row, relative to the hop's k_begin
    int64_t lim = hp.k_len;
    const int64_t qpos = pos_of(hp.q_map, valid ? row : (q_end - 1 > row0 ? q_end - 1 : row0));
    if (hp.causal) {
      int64_t cnt = count_le(hp.k_map, hp.n_k, pos_of(hp.q_map, valid ? row : q_end - 1)) -
                    hp.k_begin;
      lim = cnt < lim ? cnt : lim;
    }
    const float c2 = p.scale_log2;
    float m_run = -INFINITY, l_run = 0.f;

    for (int u = first, jj = 0; u < nu; u = next_live(u + 1), ++jj) {
      const int j = tile_at(u);
      const int64_t nvalid = lim - (int64_t)j * BN;
      uint64_t gk0 = 0, gk1 = 0;   // block-sparse grid: hidden key columns of this row
      if (kGrid && hp.grid_skip && !(use_bits && ((full_bits[j >> 5] >> (j & 31)) & 1u))) {
        // (computed before the S wait so the table lookups overlap the MMA)
        const int nv = nvalid > BN ? BN : (nvalid < 0 ? 0 : (int)nvalid);
        const int64_t kt0 = hp.k_begin + (int64_t)j * BN;
        if (nv > 0) gk0 = grid_key_bits(hp, qpos, kt0, nv < 64 ? nv : 64);
        if (nv > 64) gk1 = grid_key_bits(hp, qpos, kt0 + 64, nv - 64);
      }
      ptx::mbar_wait(s_full + g, jj & 1); FTRACE(3 + 8 * g, jj);
      ptx::tc_fence_after();
      float s[BN];
      {
        uint32_t r[BN];
#pragma unroll
        for (int cc = 0; cc < BN / 32; ++cc)
          ptx::tmem_ld32(tS + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(r + cc * 32));
        ptx::tmem_wait_ld();
        ptx::reg_fence(r);
#pragma unroll
        for (int i = 0; i < BN; ++i) s[i] = __uint_as_float(r[i]);
      }
      const bool partial = __any_sync(0xffffffffu, nvalid < BN || (gk0 | gk1) != 0);
      if (partial) {
#pragma unroll
        for (int i = 0; i < BN; ++i)
          if (i >= nvalid || (((i < 64 ? gk0 : gk1) >> (i & 63)) & 1)) s[i] = -INFINITY;
      }
      // row max as 8 independent chains (a single chain is 128 dependent FMNMX)
      float mx8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mx8[u] = s[u];
#pragma unroll
      for (int i = 8; i < BN; ++i) mx8[i & 7] = fmaxf(mx8[i & 7], s[i]);
      const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                             fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      const float m_tile = mx * c2; FTRACE(4 + 8 * g, jj);
      const bool grow = m_tile > m_run + kRescaleThreshold || (m_run == -INFINITY && m_tile > -INFINITY);
      if (__any_sync(0xffffffffu, grow && jj > 0)) {
        const float m_new = grow ? fmaxf(m_tile, m_run) : m_run;
        const float alpha = (m_run == -INFINITY) ? 0.f : ptx::ex2(m_run - m_new);
#pragma unroll
        for (int cc = 0; cc < D / 32; ++cc) {
          uint32_t r[32];
          ptx::tmem_ld32(tO + cc * 32, r);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
          ptx::tmem_st32(tO + cc * 32, r);
        }
        l_run *= alpha;
        m_run = m_new;
      } else if (grow) {
        m_run = fmaxf(m_tile, m_run);
      }
      const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
      // x = S * scale*log2e - m and the row sum on packed fp32x2 (FFMA2 / FADD2)
      float2 ls4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                       make_float2(0.f, 0.f)};
      const float2 c2v = make_float2(c2, c2), negm = make_float2(-m_use, -m_use);
      // part of the row's exp2 on the FMA pipe (ex2_poly) when no entry of the warp's
      // tile is masked; masked (-inf) entries must stay exactly 0 -> MUFU only
      // the exp loop is instantiated twice (hoisted branch): with the FMA-pipe exp2 share
      // when no entry of the warp's tile is masked, MUFU only otherwise
      auto exp_row = [&](auto use_poly) {
#pragma unroll
        for (int cc = 0; cc < kPS; ++cc) {
          constexpr int kPairs = BN / 2 / kPS;
          uint32_t pk[kPairs];
#pragma unroll
          for (int i = 0; i < kPairs; ++i) {
            const float2 x = ptx::ffma2(make_float2(s[cc * 2 * kPairs + 2 * i], s[cc * 2 * kPairs + 2 * i + 1]),
                                        c2v, negm);
            float p0, p1;
            if (decltype(use_poly)::value && (i % kPolyMod) < kPolyCnt) {
              const float2 pp = ptx::ex2_poly2(x);
              p0 = pp.x;
              p1 = pp.y;
            } else {
              p0 = ptx::ex2(x.x);
              p1 = ptx::ex2(x.y);
            }
            ls4[i & 3] = ptx::fadd2(ls4[i & 3], make_float2(p0, p1));
            pk[i] = ptx::pack_bf16(p0, p1);
          }
          if constexpr (kPairs == 64) {
            ptx::tmem_st32(tS, *reinterpret_cast<const uint32_t(*)[32]>(pk));
            ptx::tmem_st32(tS + 32, *reinterpret_cast<const uint32_t(*)[32]>(pk + 32));
          } else if constexpr (kPairs == 32) {
            ptx::tmem_st32(tS + cc * 32, *reinterpret_cast<const uint32_t(*)[32]>(pk));
          } else {
            ptx::tmem_st16(tS + cc * 16, *reinterpret_cast<const uint32_t(*)[16]>(pk));
          }
          // P for this key chunk is in TMEM: its O += P V MMAs may start
          ptx::tmem_wait_st();
          ptx::tc_fence_before();
          ptx::mbar_arrive(p_full + kPS * g + cc);
        }
      };
      if (kPolyCnt > 0 && !partial)
        exp_row(std::integral_constant<bool, kPolyCnt != 0>());
      else
        exp_row(std::integral_constant<bool, false>());
      const float2 lsa = ptx::fadd2(ptx::fadd2(ls4[0], ls4[1]), ptx::fadd2(ls4[2], ls4[3]));
      l_run += lsa.x + lsa.y;
      FTRACE(5 + 8 * g, jj);
    }

    // ------------------------------------------------------------ epilogue
    if (any) {
      ptx::mbar_wait(o_full, 0);
      ptx::tc_fence_after();
    }
    const int64_t bh = (int64_t)b * hp.heads + h;
    const int64_t NT = ceil_div(hp.n_q, 128);
    float m_old = -INFINITY, l_old = 0.f;
    if (valid && !p.first_hop) {
      m_old = p.m_run[bh * hp.n_q + row];
      l_old = p.l_run[bh * hp.n_q + row];
    }
    const float m_new = fmaxf(m_old, m_run);
    const float a_old = (m_old == -INFINITY) ? 0.f : ptx::ex2(m_old - m_new);
    const float a_hop = (m_run == -INFINITY) ? 0.f : ptx::ex2(m_run - m_new);
    const float l_new = a_old * l_old + a_hop * l_run;
    const float inv_l = (l_new > 0.f) ? 1.f / l_new : 0.f;
    // MaskError (bit 0): a row with no visible key; NonFiniteError (bit 1): a non-finite
    // O or lse (PartialAttn.finalize, local_attn.py:127-135).  `nf` turns NaN iff any
    // output value is non-finite (x * 0 = NaN for x = +-inf or NaN).
    float nf = 0.f;
    if (valid && p.finalize && l_new == 0.f) atomicOr(p.flags, 1);
#pragma unroll
    for (int cc = 0; cc < D / 32; ++cc) {
      uint32_t r[32];
      if (any) {
        ptx::tmem_ld32(tO + cc * 32, r);
        ptx::tmem_wait_ld();
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = 0u;
      }
      if (!valid) continue;
      float o[32];
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        float4 prev = make_float4(0.f, 0.f, 0.f, 0.f);
        const size_t ti = tl_index(bh, row, cc * 32 + i, D, NT);
        if (!p.first_hop) prev = *reinterpret_cast<const float4*>(p.o_acc + ti);
        o[i + 0] = a_old * prev.x + a_hop * __uint_as_float(r[i + 0]);
        o[i + 1] = a_old * prev.y + a_hop * __uint_as_float(r[i + 1]);
        o[i + 2] = a_old * prev.z + a_hop * __uint_as_float(r[i + 2]);
        o[i + 3] = a_old * prev.w + a_hop * __uint_as_float(r[i + 3]);
        if (!p.finalize)
          *reinterpret_cast<float4*>(p.o_acc + ti) = make_float4(o[i], o[i + 1], o[i + 2], o[i + 3]);
      }
      if (p.finalize) {
        __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.o_out) +
                             (((int64_t)b * hp.n_q + row) * hp.heads + h) * D + cc * 32;
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 w;
#pragma unroll
          for (int e = 0; e < 8; ++e) nf = fmaf(o[i + e] * inv_l, 0.f, nf);
          w.x = ptx::pack_bf16(o[i + 0] * inv_l, o[i + 1] * inv_l);
          w.y = ptx::pack_bf16(o[i + 2] * inv_l, o[i + 3] * inv_l);
          w.z = ptx::pack_bf16(o[i + 4] * inv_l, o[i + 5] * inv_l);
          w.w = ptx::pack_bf16(o[i + 6] * inv_l, o[i + 7] * inv_l);
          *reinterpret_cast<uint4*>(out + i) = w;
        }
      }
    }
    if (valid) {
      if (p.finalize) {
        const float lse = (l_new > 0.f) ? (m_new + __log2f(l_new)) * kLn2 : -INFINITY;
        p.lse_out[bh * hp.n_q + row] = lse;
        if (l_new != 0.f && !(fabsf(nf + lse) <= 3.0e38f)) atomicOr(p.flags, 2);
      } else {
        p.m_run[bh * hp.n_q + row] = m_new;
        p.l_run[bh * hp.n_q + row] = l_new;
      }
    }
  }

  __syncwarp();
  ptx::tc_fence_before();
  if (kPair)
    ptx::cluster_sync();   // no multicast load or remote arrive may target an exited CTA
  else
    __syncthreads();
  if (warp == 8) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tbase, 512);
  }
}

}  // namespace fwd
}  // namespace burst
