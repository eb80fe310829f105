// LAO backward on sm_100a, K/V-stationary, 16 warps: the P/dS work of a
// 128-key x 128-query step is split by query half over TWO warpgroups.
//
// Reference semantics: one call = ring.backward_step (ring.py:221-242) for every
// (batch, head) slice, i.e. local_backward (local_attn.py:255-289, tiled form
// _backward_tiled 313-353) over the hop's rectangle:
//     P = exp(S - lse); dV += P^T dO; dP = dO V^T; dS = P * (dP - D);
//     dQ += scale dS K;  dK += scale dS^T Q
// computed transposed per key tile (S^T = K Q^T): the visiting block's dK/dV
// accumulate in TMEM across all query tiles, dQ (pinned on this rank) is reduced
// into an fp32 workspace with TMA bulk reductions.
//
// Why this shape (measured on lao_bwd3, exp/trace_bwd.py): with ONE P/dS
// warpgroup (one warp per SM sub-partition) the exp phase took ~2000 cycles and
// the dS phase ~1000 of a ~4800-cycle step, both on the MMA dependency chain.
// Two warpgroups (two warps per sub-partition, 64 query columns each) halve both
// phases; the dQ drain double-buffers its SMEM staging in 16 KB quarters so the
// staging writes overlap the bulk reduction reads; the MMA issuer no longer
// blocks dK/dQ behind a late Q_{i+1} load.
//
// CTA = one key tile of 128 rows (K, V stationary in SMEM); loops over the
// hop's query tiles of 128 (Q_i + lse/D double-buffered, dO_i single-buffered).
//   warps 0-3   P/dS, query columns [0,64)   (thread = key row = TMEM lane); dV epilogue
//   warps 4-7   P/dS, query columns [64,128)                                ; dK epilogue
//   warps 8-11  dQ drain (thread = query row of the dQ tile)
//   warp  12    TMA producer (+ TMEM allocator);  warp 13 tcgen05.mma issuer
// TMEM (512 cols for D=128): S^T [0,128) with P^T (bf16) of query half h written
// over S^T columns [64h, 64h+32) by the warpgroup that read them; dP^T [128,256), with
// dS^T (bf16, the A operand of dK) written the same way over [128+64h, +32), then dQ_i
// once dK_i has read it; dV [256,256+D); dK [256+D,256+2D).
#pragma once
#include <cuda.h>
#include "common.cuh"
#include "ptx.cuh"

namespace burst {
namespace bwd4 {

#ifndef BURST_BWD_ROT   // query-tile rotation multiplier per walker (CTA or cluster)
#define BURST_BWD_ROT 7
#endif

constexpr int BM = 128;  // query rows per iteration
constexpr int BN = 128;  // key rows per CTA
constexpr int kThreads = 512;

template <int D>
struct Cfg {
  static constexpr int kBoxBytes = 128 * 64 * 2;
  static constexpr int kBoxes = D / 64;
  static constexpr int kTileBytes = kBoxBytes * kBoxes;    // K, V, Q_i, dO_i tiles
  static constexpr int kDsBytes = BN * BM * 2;              // dS^T tile (bf16)
  static constexpr int kStatBytes = 2 * BM * 4;             // lse2_i, D_i
  static constexpr int kQuarterBytes = BM * 32 * 4;         // dQ staging: 32 columns
  static constexpr int kPayload = 2 * kTileBytes + 2 * kTileBytes + kTileBytes + kDsBytes +
                                  2 * kQuarterBytes + 2 * kStatBytes;
  static constexpr int kLiveWords = 64;    // live-query-tile bitmap (grid masks): 2048 tiles
  static constexpr int kBarBytes = 136 + 4 * kLiveWords;
  static constexpr int kMaxSmem = 232448;
  static constexpr int kSmemBytes =
      (kPayload + kBarBytes + 1024 <= kMaxSmem) ? kPayload + kBarBytes + 1024 : kMaxSmem;
  static constexpr int kMaxPad = kSmemBytes - kPayload - kBarBytes;
};

struct Params {
  CUtensorMap tm_q, tm_k, tm_v, tm_do;
  CUtensorMap tm_q64, tm_do64;   // 64-row boxes (clusters of 4)
  const float* stats;    // [2][B*H][NTq*128]: lse*log2e, D
  float* dq_acc;         // TL over n_q
  float* dk_acc;         // TL over n_k
  float* dv_acc;
  burst_hop hop;
  float scale_log2, scale;
  int accumulate;
  long long* trace;   // BURST_TRACE builds only: per-iteration clock64 timeline
  unsigned long long* life;   // BURST_LIFE builds only: per-CTA globaltimer events
};

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          ptx::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(ptx::smem_u32(bar))
      : "memory");
}

#ifdef BURST_TRACE
#define BTRACE4(ev, i)                                                                       \
  do {                                                                                       \
    if (p.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (i) < 64)       \
      p.trace[(ev) * 64 + (i)] = clock64();                                                  \
  } while (0)
#else
#define BTRACE4(ev, i)
#endif
#ifdef BURST_LIFE   // experiment: CTA lifetime events (globaltimer ns; slot 7 = SM id)
#define BLIFE(ev)                                                                            \
  do {                                                                                       \
    unsigned long long t_;                                                                   \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                   \
    const size_t c_ = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x; \
    if (p.life && c_ < 65536) p.life[c_ * 16 + (ev)] = t_;                                    \
    if ((ev) == 0 && p.life && c_ < 65536) {                                                 \
      unsigned s_; asm volatile("mov.u32 %0, %%smid;" : "=r"(s_)); p.life[c_ * 16 + 7] = s_;  \
    }                                                                                        \
  } while (0)
#else
#define BLIFE(ev)
#endif

// kGrid: the hop carries a block-sparse grid mask (tile skipping + element masks);
// the instantiation without it keeps the dense loops free of the skip bookkeeping.
// kOrdered: deterministic mode (p.dq_order set) -- dK/dV only; dQ is computed by the
// query-stationary lao_dq kernel (lao_dq_sm100.cuh), one writer per dQ row, so no
// order-dependent fp32 reduction remains.  The dS SMEM stores, the dQ MMA and the
// drain are compiled out; dP^T_{i+1} waits for dK_i (the last reader of dS^T).
// kCl (cluster size 1, 2 or 4): launched as kCl-CTA clusters over consecutive key tiles
// that walk the SAME query tiles; each CTA TMA-loads 1/kCl of every Q and dO tile (a
// 64-column box, or a 64-row half of one for kCl = 4) and multicasts it to all (1/kCl
// of the L2 reads of Q/dO, which are ~40% of the unclustered backward's L2 traffic); a
// stage is refilled only once every CTA has released it (kCl-count empty barriers fed
// by multicast MMA commits).
template <int D, bool kGrid, bool kOrdered, int kCl = 1>
__global__ void __launch_bounds__(kThreads, 1) lao_bwd4_kernel(const __grid_constant__ Params p) {
  using C = Cfg<D>;
  static_assert(kCl == 1 || D == 128, "clustered backward splits Q/dO tiles by 64-column box");
  static_assert(kCl == 1 || kCl == 2 || kCl == 4, "cluster of 1, 2 or 4 CTAs");
  constexpr bool kPair = kCl > 1;
  constexpr uint16_t kMask = (uint16_t)((1u << kCl) - 1u);
  // SW128 tiles need 1024-byte alignment; the declaration asks the compiler for it and
  // the runtime check below can then only fail on a toolchain that ignores it, in
  // which case the launch reports a CudaError (flag bit 2) instead of trapping.
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (threadIdx.x == 0) BLIFE(0);
  uint8_t* smem;
  {
    const uint32_t s = ptx::smem_u32(smem_raw);
    const uint32_t pad = (1024u - (s & 1023u)) & 1023u;
    if (pad > (uint32_t)C::kMaxPad) {
      if (threadIdx.x == 0 && p.hop.flags) atomicOr(p.hop.flags, 4);
      return;
    }
    smem = smem_raw + pad;
  }
  uint8_t* sK = smem;
  uint8_t* sV = sK + C::kTileBytes;
  uint8_t* sQ = sV + C::kTileBytes;            // [2] stages
  uint8_t* sdO = sQ + 2 * C::kTileBytes;       // single buffer
  uint8_t* sdS = sdO + C::kTileBytes;
  float* sStage = reinterpret_cast<float*>(sdS + C::kDsBytes);  // [2] x [8][128] float4
  float* sStat = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(sStage) + 2 * C::kQuarterBytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sStat) + 2 * C::kStatBytes);
  uint64_t* kv_full = bars;
  uint64_t* qdo_full = bars + 1;   // [2]
  uint64_t* qdo_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;
  uint64_t* p_full = bars + 6;
  uint64_t* ds_full = bars + 7;
  uint64_t* ds_empty = bars + 8;
  uint64_t* dq_full = bars + 9;
  uint64_t* dq_empty = bars + 10;
  uint64_t* dkv_full = bars + 11;
  uint64_t* dp_full = bars + 12;
  uint64_t* do_full = bars + 13;
  uint64_t* do_empty = bars + 14;
  uint64_t* dst_full = bars + 15;   // dS^T in TMEM (dK may start; dS still on its way to SMEM)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 16);

  const burst_hop& hp = p.hop;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.z, h = blockIdx.y;
  const int64_t bh = (int64_t)b * hp.heads + h;
  const int64_t k0 = hp.k_begin + (int64_t)blockIdx.x * BN;   // first key row of this CTA
  const int64_t k_end = hp.k_begin + hp.k_len;
  // the key rows whose query walk this CTA follows: its own, or its cluster pair's 256
  const uint32_t crank = kPair ? ptx::cluster_rank() : 0u;
  const int64_t kw0 = hp.k_begin + (int64_t)(blockIdx.x & ~(unsigned)(kCl - 1)) * BN;
  const int64_t kwrows = (kw0 + kCl * BN < k_end ? kw0 + kCl * BN : k_end) - kw0;
  const int64_t q_end = hp.q_begin + hp.q_len;
  const int64_t NTq = ceil_div(hp.n_q, 128);
  const int64_t NTk = ceil_div(hp.n_k, 128);

  // Query tiles touching this key tile, on the block's absolute 128-row grid (so every
  // dQ tile is one contiguous TL run): causal => a suffix of the hop's queries.  Rows
  // of the first tile before q_begin (unaligned zigzag chunks) or before the causal
  // frontier are masked like causal columns.
  int64_t qlo = hp.q_begin;
  if (hp.causal) {
    const int64_t first_q = count_le(hp.q_map, hp.n_q, pos_of(hp.k_map, kw0) - 1);
    if (first_q > qlo) qlo = first_q;
  }
  const int64_t qs = (qlo / BM) * BM;
  const int nq = qs < q_end ? (int)ceil_div(q_end - qs, BM) : 0;
  // Query-tile order rotated per CTA: concurrently resident CTAs (consecutive key
  // tiles of one head) reduce into different dQ tiles (measured best at 128K,
  // profiles/r01_rotation_exp.txt).
  const unsigned walker = blockIdx.x / kCl;
  const int rot = nq > 0 ? (int)((walker * (unsigned)BURST_BWD_ROT) % (unsigned)nq) : 0;
  auto qtile = [&](int i) -> int64_t { int j = i + rot; if (j >= nq) j -= nq; return qs + (int64_t)j * BM; };
  // Block-sparse grid: query tiles whose every (query, key) pair with this CTA's keys
  // lies in skipped cells are skipped by every role.  Roles count LIVE tiles (stages,
  // barrier parities); the producer, P/dS and drain map them back to tile indices.
  auto live = [&](int i) -> bool {   // (kPair: live for either CTA of the pair)
    if (!kGrid) return true;
    const int64_t q0 = qtile(i) < hp.q_begin ? hp.q_begin : qtile(i);
    return grid_rect_live(hp, q0, (qtile(i) + BM < q_end ? qtile(i) + BM : q_end) - q0, kw0, kwrows);
  };
  // The predicate is evaluated once per tile by the whole CTA into a SMEM bitmap (up to
  // kLiveWords * 32 tiles); every role then finds the next live tile with __ffs.
  uint32_t* live_bits = tmem_holder + 2;
  const bool use_bits = kGrid && nq <= C::kLiveWords * 32;
  auto next_live = [&](int i) -> int {
    if (!kGrid) return i;
    if (use_bits) {
      if (i >= nq) return nq;
      int w = i >> 5;
      uint32_t m = live_bits[w] & (~0u << (i & 31));
      const int nw = (nq + 31) >> 5;
      while (m == 0u) {
        if (++w >= nw) return nq;
        m = live_bits[w];
      }
      const int r = (w << 5) + __ffs(m) - 1;
      return r < nq ? r : nq;
    }
    while (i < nq && !live(i)) ++i;
    return i;
  };
  int nlive = nq;   // kGrid: counted cooperatively by the whole CTA below

  if (warp == 12) {
    if (lane == 0) {
      ptx::mbar_init(kv_full, 1);
      for (int s = 0; s < 2; ++s) {
        ptx::mbar_init(qdo_full + s, 1);
        ptx::mbar_init(qdo_empty + s, kCl);
      }
      ptx::mbar_init(s_full, 1);
      ptx::mbar_init(p_full, 2 * BN);
      ptx::mbar_init(ds_full, 2 * BN);
      ptx::mbar_init(dst_full, 2 * BN);
      ptx::mbar_init(ds_empty, 1);
      ptx::mbar_init(dq_full, 1);
      ptx::mbar_init(dq_empty, BM);
      ptx::mbar_init(dkv_full, 1);
      ptx::mbar_init(dp_full, 1);
      ptx::mbar_init(do_full, 1);
      ptx::mbar_init(do_empty, kCl);
      ptx::fence_mbar_init();
      ptx::tma_prefetch_desc(&p.tm_q);
      ptx::tma_prefetch_desc(&p.tm_k);
      ptx::tma_prefetch_desc(&p.tm_v);
      ptx::tma_prefetch_desc(&p.tm_do);
    }
    __syncwarp();
    ptx::tmem_alloc(tmem_holder, 512);
  }
  if (kGrid) {
    if (threadIdx.x == 0) tmem_holder[1] = 0;
    if (use_bits)
      for (int w = threadIdx.x; w < ((nq + 31) >> 5); w += kThreads) live_bits[w] = 0u;
    __syncthreads();
    int mine = 0;
    for (int i = threadIdx.x; i < nq; i += kThreads) {
      const bool l = live(i);
      mine += l ? 1 : 0;
      if (l && use_bits) atomicOr(live_bits + (i >> 5), 1u << (i & 31));
    }
    mine = __reduce_add_sync(0xffffffffu, mine);
    if (lane == 0 && mine) atomicAdd(tmem_holder + 1, (uint32_t)mine);
  }
  ptx::tc_fence_before();
  if (kPair)
    ptx::cluster_sync();   // both CTAs' barriers exist before either multicasts into them
  else
    __syncthreads();
  ptx::tc_fence_after();
  if (threadIdx.x == 0) BLIFE(1);
  const uint32_t tbase = *tmem_holder;
  if (kGrid) nlive = (int)tmem_holder[1];
  constexpr uint32_t kS = 0, kDP = 128, kDV = 256, kDK = 256 + D;
  if (warp >= 12) {
   ptx::regs_dec<80>();
#ifdef BURST_TRACE
   if (warp == 14 && lane == 0 && blockIdx.x == 0) {
     // observer: completion times of the MMA groups (tensor-pipe timeline)
     for (int i = 0; i < nlive && i < 64; ++i) {
       ptx::mbar_wait(s_full, i & 1); BTRACE4(16, i);
       ptx::mbar_wait(do_empty, i & 1); BTRACE4(17, i);     // dV_i done
       ptx::mbar_wait(dq_full, i & 1); BTRACE4(18, i);      // dK_i, dQ_i done
       if (i + 1 < nlive) { ptx::mbar_wait(dp_full, (i + 1) & 1); BTRACE4(19, i); }   // dP^T_{i+1} done
     }
   }
#endif
   if (warp == 12) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && nlive > 0) {
      ptx::mbar_expect_tx(kv_full, 2 * C::kTileBytes);
      for (int x = 0; x < C::kBoxes; ++x) {
        ptx::tma_load_4d(sK + x * C::kBoxBytes, &p.tm_k, kv_full, x * 64, h, (int)k0, b);
        ptx::tma_load_4d(sV + x * C::kBoxBytes, &p.tm_v, kv_full, x * 64, h, (int)k0, b);
      }
      auto load_q = [&](int j, int ti) {   // j = live index, ti = query tile index
        const int s = j & 1;
        const int64_t q0 = qtile(ti);
        ptx::mbar_wait(qdo_empty + s, ((j >> 1) & 1) ^ 1);
        ptx::mbar_expect_tx(qdo_full + s, C::kTileBytes + C::kStatBytes);
        if (kCl == 2)
          ptx::tma_load_4d_mc(sQ + s * C::kTileBytes + crank * C::kBoxBytes, &p.tm_q, qdo_full + s,
                              (int)crank * 64, h, (int)q0, b, kMask);
        else if (kCl == 4)   // 64-row half (crank >> 1) of column box (crank & 1)
          ptx::tma_load_4d_mc(sQ + s * C::kTileBytes + (crank & 1) * C::kBoxBytes + (crank >> 1) * 8192,
                              &p.tm_q64, qdo_full + s, (int)(crank & 1) * 64, h,
                              (int)(q0 + (crank >> 1) * 64), b, kMask);
        else
          for (int x = 0; x < C::kBoxes; ++x)
            ptx::tma_load_4d(sQ + s * C::kTileBytes + x * C::kBoxBytes, &p.tm_q, qdo_full + s,
                             x * 64, h, (int)q0, b);
        const float* st = p.stats + bh * NTq * 128 + q0;
        bulk_load(sStat + s * 2 * BM, st, BM * 4, qdo_full + s);
        bulk_load(sStat + s * 2 * BM + BM, st + (int64_t)hp.batch * hp.heads * NTq * 128, BM * 4,
                  qdo_full + s);
      };
      auto load_do = [&](int j, int ti) {
        ptx::mbar_wait(do_empty, (j & 1) ^ 1);
        ptx::mbar_expect_tx(do_full, C::kTileBytes);
        if (kCl == 2)
          ptx::tma_load_4d_mc(sdO + crank * C::kBoxBytes, &p.tm_do, do_full, (int)crank * 64, h,
                              (int)qtile(ti), b, kMask);
        else if (kCl == 4)
          ptx::tma_load_4d_mc(sdO + (crank & 1) * C::kBoxBytes + (crank >> 1) * 8192, &p.tm_do64,
                              do_full, (int)(crank & 1) * 64, h, (int)(qtile(ti) + (crank >> 1) * 64),
                              b, kMask);
        else
          for (int x = 0; x < C::kBoxes; ++x)
            ptx::tma_load_4d(sdO + x * C::kBoxBytes, &p.tm_do, do_full, x * 64, h, (int)qtile(ti), b);
      };
      int tq = next_live(0), td = tq;      // next tile of the Q and of the dO load stream
      load_q(0, tq); tq = next_live(tq + 1);
      load_do(0, td); td = next_live(td + 1);
      if (nlive > 1) { load_q(1, tq); tq = next_live(tq + 1); }
      for (int i = 0; i < nlive; ++i) {      // release order: dO after dV_i, Q stage after dK_i
        if (i + 1 < nlive) { load_do(i + 1, td); td = next_live(td + 1); }
        if (i + 2 < nlive) { load_q(i + 2, tq); tq = next_live(tq + 1); }
      }
    }
   } else if (warp == 13) {
    // ------------------------------------------------------------ MMA issuer
    // Per query tile i: dV_i | {S^T_{i+1}, dK_i + dQ_i -> dP region} in whichever
    // order their inputs arrive (S^T first when both are ready) | dP^T_{i+1} once
    // dQ_i has been drained to registers.  The whole warp runs the loop (uniform
    // control flow keeps descriptors in uniform registers); one elected lane issues
    // each MMA group and its commits.  Descriptors: base + (byte offset >> 4).
    if (nlive > 0) {
      constexpr uint32_t id_kk = ptx::make_idesc_bf16(BN, BM, 0, 0);   // S^T, dP^T
      constexpr uint32_t id_kmn = ptx::make_idesc_bf16(BN, D, 0, 1);   // dV, dK (B MN-major)
      constexpr uint32_t id_mnmn = ptx::make_idesc_bf16(BM, D, 1, 1);  // dQ (A, B MN-major)
      const uint64_t dK = ptx::make_sdesc(ptx::smem_u32(sK), 0, 1024);
      const uint64_t dV = ptx::make_sdesc(ptx::smem_u32(sV), 0, 1024);
      const uint64_t dQ0 = ptx::make_sdesc(ptx::smem_u32(sQ), 0, 1024);
      const uint64_t dOk = ptx::make_sdesc(ptx::smem_u32(sdO), 0, 1024);           // K-major (dP^T)
      const uint64_t dOm = ptx::make_sdesc(ptx::smem_u32(sdO), C::kBoxBytes, 1024); // MN-major (dV)
      const uint64_t dQm0 = ptx::make_sdesc(ptx::smem_u32(sQ), C::kBoxBytes, 1024); // MN-major (dK)
      const uint64_t dSm = ptx::make_sdesc(ptx::smem_u32(sdS), 16384, 1024);       // dS MN-major (dQ)
      const uint64_t dKm = ptx::make_sdesc(ptx::smem_u32(sK), C::kBoxBytes, 1024);  // K MN-major (dQ)
      constexpr uint64_t kStage = (uint64_t)(C::kTileBytes >> 4);
      auto kmaj = [](int kk) -> uint64_t { return (uint64_t)(((kk >> 2) * C::kBoxBytes + (kk & 3) * 32) >> 4); };
      auto st_mma = [&](int stage) {   // S^T = K Q^T
        if (ptx::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            ptx::mma_ss(tbase + kS, dK + kmaj(kk), dQ0 + stage * kStage + kmaj(kk), id_kk, kk > 0);
          ptx::mma_commit(s_full);
        }
        __syncwarp();
      };
      auto dpt_mma = [&]() {  // dP^T = V dO^T
        if (ptx::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            ptx::mma_ss(tbase + kDP, dV + kmaj(kk), dOk + kmaj(kk), id_kk, kk > 0);
          ptx::mma_commit(dp_full);
        }
        __syncwarp();
      };
      auto dk_mma = [&](int i) {   // dK += dS^T Q (A = dS^T in TMEM); last reader of Q_i
        if (ptx::elect_one()) {
          const uint64_t qm = dQm0 + (i & 1) * kStage;
#pragma unroll
          for (int kk = 0; kk < BM / 16; ++kk)
            // A = dS^T from TMEM; the dQ MMAs below overwrite those columns, and in-order
            // execution of one thread's MMAs keeps that after this read
            ptx::mma_ts(tbase + kDK, tbase + kDP + (kk < 4 ? kk * 8 : 32 + kk * 8),
                        qm + (uint64_t)(kk * 2048 >> 4), id_kmn, (i > 0 || kk > 0) ? 1u : 0u);
          if (kPair)
            ptx::mma_commit_mc(qdo_empty + (i & 1), kMask);   // this CTA released the stage, in all
          else
            ptx::mma_commit(qdo_empty + (i & 1));
          if (kOrdered) ptx::mma_commit(dq_full);   // dS^T read: the dP^T columns are free
        }
        __syncwarp();
      };
      auto dq_mma = [&]() {   // dQ_i = dS K into the dP^T columns (issued after dK_i read them)
        if (ptx::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk)
            ptx::mma_ss(tbase + kDP, dSm + (uint64_t)(kk * 2048 >> 4), dKm + (uint64_t)(kk * 2048 >> 4),
                        id_mnmn, kk > 0);
          ptx::mma_commit(dq_full);
          ptx::mma_commit(ds_empty);
        }
        __syncwarp();
      };
      ptx::mbar_wait(kv_full, 0);
      ptx::mbar_wait(qdo_full + 0, 0);
      ptx::tc_fence_after();
      st_mma(0);
      ptx::mbar_wait(do_full, 0);
      ptx::tc_fence_after();
      dpt_mma();
      for (int i = 0; i < nlive; ++i) {
        const int s = i & 1;
        const bool more = i + 1 < nlive;
        // dV += P^T dO   (A = P^T from TMEM: query half h at S^T columns [64h, 64h+32))
        ptx::mbar_wait(p_full, i & 1); BTRACE4(0, i);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BM / 16; ++kk)
            ptx::mma_ts(tbase + kDV, tbase + kS + (kk < 4 ? kk * 8 : 32 + kk * 8),
                        dOm + (uint64_t)(kk * 2048 >> 4), id_kmn, (i > 0 || kk > 0) ? 1u : 0u);
          if (kPair)
            ptx::mma_commit_mc(do_empty, kMask);
          else
            ptx::mma_commit(do_empty);
        }
        __syncwarp();
        bool st_done = !more, dk_done = false, dq_done = false;
        while (!st_done || !dq_done) {
          if (!st_done && ptx::mbar_try_wait(qdo_full + (s ^ 1), ((i + 1) >> 1) & 1)) {
            BTRACE4(11, i);
            ptx::tc_fence_after();
            st_mma(s ^ 1);
            st_done = true;
          }
          if (!dk_done && ptx::mbar_try_wait(dst_full, i & 1)) {
            ptx::tc_fence_after();
            dk_mma(i);
            dk_done = true;
            if (kOrdered) dq_done = true;
          }
          if (dk_done && !dq_done && ptx::mbar_try_wait(ds_full, i & 1)) {
            BTRACE4(1, i);
            ptx::tc_fence_after();
            dq_mma();
            dq_done = true;
          }
        }
        if (more) {
          ptx::mbar_wait(kOrdered ? dq_full : dq_empty, i & 1); BTRACE4(2, i);
          ptx::mbar_wait(do_full, (i + 1) & 1); BTRACE4(10, i);
          ptx::tc_fence_after();
          dpt_mma();
        }
      }
      if (ptx::elect_one()) ptx::mma_commit(dkv_full);
      __syncwarp();
    }
   }
  } else if (warp < 8) {
    // ------------------------------------------------------------ P / dS, query half hq
    ptx::regs_inc<144>();
    const int hq = warp >> 2;                   // query columns [64 hq, 64 hq + 64)
    const int t = threadIdx.x & 127;            // key row within the tile
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int64_t krow = k0 + t;
    const bool kvalid = krow < k_end && krow < hp.n_k;
    const int64_t kpos = (hp.causal || kGrid) ? pos_of(hp.k_map, kvalid ? krow : k0) : 0;
    int64_t qfirst = hp.causal ? count_le(hp.q_map, hp.n_q, kpos - 1) : 0;
    if (qfirst < hp.q_begin) qfirst = hp.q_begin;
    const float c2 = p.scale_log2;
    for (int i = 0, ti = next_live(0); i < nlive; ++i, ti = next_live(ti + 1)) {
      const int s = i & 1;
      const int64_t q0 = qtile(ti) + 64 * hq;
      // visible query columns of this key row within the half: [lo, hi)
      int64_t lo64 = qfirst - q0, hi64 = q_end - q0;
      const int lo = lo64 < 0 ? 0 : (lo64 > 64 ? 64 : (int)lo64);
      const int hi = !kvalid ? 0 : (hi64 > 64 ? 64 : (hi64 < 0 ? 0 : (int)hi64));
      uint64_t gq = 0;   // block-sparse grid: hidden query columns of this half
      if (kGrid) {
        const int nv = hi64 > 64 ? 64 : (hi64 < 0 ? 0 : (int)hi64);
        if (nv > 0) gq = grid_query_bits(hp, q0, nv, kpos);
      }
      const bool warp_full = __all_sync(0xffffffffu, lo == 0 && hi == 64 && gq == 0);
      ptx::mbar_wait(qdo_full + s, (i >> 1) & 1);
      ptx::mbar_wait(s_full, i & 1); if (hq == 0) BTRACE4(3, i);
      if (i == 0 && threadIdx.x == 0) BLIFE(2);
      ptx::tc_fence_after();
      const float4* lse4 = reinterpret_cast<const float4*>(sStat + s * 2 * BM) + 16 * hq;
      const float4* dst4 = lse4 + BM / 4;
      float pr[64];
      {
        uint32_t r[64];
        ptx::tmem_ld32(tbase + lane_off + kS + 64 * hq, *reinterpret_cast<uint32_t(*)[32]>(r));
        ptx::tmem_ld32(tbase + lane_off + kS + 64 * hq + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
        ptx::tmem_wait_ld();
        ptx::reg_fence(r);
        if (hq == 0) BTRACE4(12, i);
#pragma unroll
        for (int c4 = 0; c4 < 16; ++c4) {
          const float4 L = lse4[c4];
          // masked entries are zeroed below, so the FMA-pipe exp2 is safe everywhere here
          // x = S * scale*log2e - lse*log2e on packed fp32x2 (FFMA2)
          const float2 xa = ptx::ffma2(make_float2(__uint_as_float(r[4 * c4 + 0]), __uint_as_float(r[4 * c4 + 1])),
                                       make_float2(c2, c2), make_float2(-L.x, -L.y));
          const float2 xb = ptx::ffma2(make_float2(__uint_as_float(r[4 * c4 + 2]), __uint_as_float(r[4 * c4 + 3])),
                                       make_float2(c2, c2), make_float2(-L.z, -L.w));
          pr[4 * c4 + 0] = ptx::ex2(xa.x);
          pr[4 * c4 + 1] = ptx::ex2(xa.y);
          pr[4 * c4 + 2] = ptx::ex2(xb.x);
          pr[4 * c4 + 3] = ptx::ex2(xb.y);
        }
      }
      if (!warp_full) {
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (c < lo || c >= hi || ((gq >> c) & 1)) pr[c] = 0.f;
      }
      {
        uint32_t pk[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) pk[j] = ptx::pack_bf16(pr[2 * j], pr[2 * j + 1]);
        if (hq == 0) BTRACE4(13, i);
        ptx::tmem_st32(tbase + lane_off + kS + 64 * hq, pk);
      }
      ptx::tmem_wait_st();
      if (hq == 0) BTRACE4(14, i);
      ptx::tc_fence_before();
      ptx::mbar_arrive(p_full); if (hq == 0) BTRACE4(4, i); else BTRACE4(22, i);

      ptx::mbar_wait(dp_full, i & 1); if (hq == 0) BTRACE4(5, i);
      if (!kOrdered) ptx::mbar_wait(ds_empty, (i & 1) ^ 1);
      ptx::tc_fence_after();
      uint8_t* rowp = sdS + hq * 16384 + t * 128;   // SW128 K-major box of this query half
      // both 32-column halves of this warpgroup's dP^T in one TMEM round trip
      uint32_t rr[64];
      ptx::tmem_ld32(tbase + lane_off + kDP + 64 * hq, *reinterpret_cast<uint32_t(*)[32]>(rr));
      ptx::tmem_ld32(tbase + lane_off + kDP + 64 * hq + 32, *reinterpret_cast<uint32_t(*)[32]>(rr + 32));
      ptx::tmem_wait_ld();
      ptx::reg_fence(rr);
      if (hq == 0) BTRACE4(20, i);
      uint32_t pks[32];   // dS of both 32-query halves, packed bf16
#pragma unroll
      for (int qc = 0; qc < 2; ++qc) {
        const uint32_t* r = rr + 32 * qc;
        uint32_t* pk = pks + 16 * qc;
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          const float4 Dv = dst4[qc * 8 + j4];
          const int c = qc * 32 + 4 * j4;
          // dS = P * (dP - D) on packed fp32x2 (FADD2 + FMUL2)
          const float2 da = ptx::fmul2(make_float2(pr[c], pr[c + 1]),
                                       ptx::fadd2(make_float2(__uint_as_float(r[4 * j4]), __uint_as_float(r[4 * j4 + 1])),
                                                  make_float2(-Dv.x, -Dv.y)));
          const float2 db = ptx::fmul2(make_float2(pr[c + 2], pr[c + 3]),
                                       ptx::fadd2(make_float2(__uint_as_float(r[4 * j4 + 2]), __uint_as_float(r[4 * j4 + 3])),
                                                  make_float2(-Dv.z, -Dv.w)));
          pk[2 * j4] = ptx::pack_bf16(da.x, da.y);
          pk[2 * j4 + 1] = ptx::pack_bf16(db.x, db.y);
        }
        // dS^T (bf16) over the dP^T columns this warpgroup has read, in the P^T layout:
        // the A operand of dK from TMEM (32 KB less SMEM read per step)
        ptx::tmem_st16(tbase + lane_off + kDP + 64 * hq + 16 * qc,
                       *reinterpret_cast<const uint32_t(*)[16]>(pk));
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive(dst_full);   // dK_i may start while dS goes to SMEM for dQ_i
      if (kOrdered) continue;       // deterministic mode: dQ comes from lao_dq
#pragma unroll
      for (int qc = 0; qc < 2; ++qc) {
        const uint32_t* pk = pks + 16 * qc;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int ch = qc * 4 + u;   // 16-byte chunk (8 queries) of the 128 B swizzle row
          *reinterpret_cast<uint4*>(rowp + ((ch ^ (t & 7)) << 4)) =
              make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
      }
      if (hq == 0) BTRACE4(21, i);
      ptx::fence_proxy_async_smem();
      ptx::tc_fence_before();
      ptx::mbar_arrive(ds_full); if (hq == 0) BTRACE4(6, i); else BTRACE4(23, i);
    }
    // -------------------------------------------------------- dK / dV epilogue
    if (nlive > 0) {
      ptx::mbar_wait(dkv_full, 0);
      ptx::tc_fence_after();
    }
    {
      float* dst = hq == 0 ? p.dv_acc : p.dk_acc;
      const float mul = hq == 0 ? 1.f : p.scale;
      const uint32_t col0 = hq == 0 ? kDV : kDK;
#pragma unroll 1
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t r[32];
        if (nlive > 0) {
          ptx::tmem_ld32(tbase + lane_off + col0 + cc * 32, r);
          ptx::tmem_wait_ld();
          ptx::reg_fence(r);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = 0u;
        }
        if (!kvalid) continue;
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float4* a = reinterpret_cast<float4*>(dst + tl_index(bh, krow, cc * 32 + j, D, NTk));
          float4 v = make_float4(__uint_as_float(r[j]) * mul, __uint_as_float(r[j + 1]) * mul,
                                 __uint_as_float(r[j + 2]) * mul, __uint_as_float(r[j + 3]) * mul);
          if (p.accumulate) {
            const float4 o = *a;
            v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
          }
          *a = v;
        }
      }
    }
  } else {
    // ------------------------------------------------------------ dQ drain (warps 8-11)
    // TMEM -> registers (whole tile, then dq_empty) -> SMEM staging in 32-column
    // quarters (two 16 KB buffers) -> one TMA bulk reduction per quarter into the TL
    // workspace (each quarter of a 128-row tile is a contiguous 16 KB run there).
    ptx::regs_inc<144>();
    const int t = threadIdx.x & 127;           // query row within the tile
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    float4* stg = reinterpret_cast<float4*>(sStage);
    for (int i = 0, ti = next_live(0); i < (kOrdered ? 0 : nlive); ++i, ti = next_live(ti + 1)) {
      const int64_t q0 = qtile(ti);
      const bool qvalid = q0 + t >= hp.q_begin && q0 + t < q_end && q0 + t < hp.n_q;
      ptx::mbar_wait(dq_full, i & 1); BTRACE4(7, i);
      ptx::tc_fence_after();
      uint32_t r[D];
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc)
        ptx::tmem_ld32(tbase + lane_off + kDP + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(r + cc * 32));
      ptx::tmem_wait_ld();
      ptx::reg_fence(r);
      ptx::tc_fence_before();
      ptx::mbar_arrive(dq_empty); BTRACE4(8, i);
      const float sc = qvalid ? p.scale : 0.f;
#if defined(BURST_EXP_DQ_REDG)    // experiment: per-thread red.global from registers
      if (qvalid) {
        float* base = p.dq_acc + tl_index(bh, q0 + t, 0, D, NTq);
#pragma unroll
        for (int j = 0; j < D; j += 4)
          ptx::red_add_v4(base + (size_t)(j >> 2) * 512, __uint_as_float(r[j]) * sc,
                          __uint_as_float(r[j + 1]) * sc, __uint_as_float(r[j + 2]) * sc,
                          __uint_as_float(r[j + 3]) * sc);
      }
      if (false)
#elif defined(BURST_EXP_NO_DQ)     // experiment: no dQ traffic at all (upper bound)
      if (false)
#endif
#pragma unroll
      for (int qq = 0; qq < D / 32; ++qq) {
        float4* buf = stg + (qq & 1) * (8 * 128);
        if (t == 0) ptx::bulk_wait_read<1>();   // the reduction that last read this buffer
        ptx::named_bar_sync(1, 128);
#ifdef BURST_EXP_NO_STAGE_STS   // experiment: staging never written (wrong results)
        if (r[qq] == 0x7f7f7f7fu)
#endif
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          const int c = qq * 32 + 4 * g;
          buf[g * 128 + t] = make_float4(__uint_as_float(r[c]) * sc, __uint_as_float(r[c + 1]) * sc,
                                         __uint_as_float(r[c + 2]) * sc, __uint_as_float(r[c + 3]) * sc);
        }
        ptx::fence_proxy_async_smem();
        ptx::named_bar_sync(1, 128);
        if (t == 0) {
          ptx::bulk_reduce_add_f32(p.dq_acc + tl_index(bh, q0, qq * 32, D, NTq), buf,
                                   C::kQuarterBytes);
          ptx::bulk_commit();
        }
      }
      BTRACE4(9, i);
    }
    if (t == 0) BLIFE(3);
    if (t == 0) ptx::bulk_wait_all();
  }

  __syncwarp();
  if (threadIdx.x == 0) BLIFE(4);
  ptx::tc_fence_before();
  if (kPair)
    ptx::cluster_sync();   // no multicast load or remote arrive may target an exited CTA
  else
    __syncthreads();
  if (threadIdx.x == 0) BLIFE(5);
  if (warp == 12) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tbase, 512);
  }
}

}  // namespace bwd4
}  // namespace burst
