// EXPERIMENT (not built; parity-green, ~1.3% slower than lao_bwd4's load-sharing pairs,
// profiles/r02_bwd_pair_experiments.txt).  Include path assumes paper_2403_09347_b200/csrc.
// LAO backward on sm_100a for CTA PAIRS with 2-SM MMAs (head_dim 128):
// lao_bwd4's pipeline, but the two CTAs of a cluster (key tiles 2p, 2p+1, walking the
// same query tiles) run S^T, dP^T, dV and dK as ONE tcgen05.mma.cta_group::2 each
// (M = 256 keys), issued by the leader, while each CTA keeps its own 1-SM dQ MMA over
// its own keys (no dS exchange).  A 2-SM MMA reads B as per-CTA halves, so every CTA
// holds only what its half needs of each Q / dO tile:
//   QR = query rows [64c, 64c+64) x all D   (B of S^T / dP^T, K-major, N split by rows)
//   QC = all 128 query rows x D cols [64c, 64c+64)   (B of dK / dV, MN-major, N split by D)
// loaded by the CTA itself with the 2-SM TMA form (completion on the leader's barrier).
// Per step an SM reads 16 KB less B for each of S^T, dP^T, dV, dK than lao_bwd4; the
// pair reads Q / dO from L2 twice (QR and QC) instead of once (multicast).
// Same math: local_backward (local_attn.py:255-353), ring.backward_step (ring.py:221-242).
//
// Cross-CTA hand-offs (leader = cluster rank 0):
//   p_full, dst_full, dq_empty live in the leader; both CTAs' warps arrive there
//   s_full, dp_full, qdo_empty, do_empty, dk_done, dkv_full: the leader's 2-SM commits
//   arrive in both CTAs (multicast)
//   each CTA's dQ_i waits dk_done (the leader's dK_i has read its dS^T in TMEM) and its
//   own ds_full; dq_full / ds_empty are local.
#pragma once
#include <cuda.h>
#include "common.cuh"
#include "ptx.cuh"
#include "lao_bwd4_sm100.cuh"

namespace burst {
namespace bwd7 {

using bwd4::BM;
using bwd4::BN;
using bwd4::kThreads;
using Params = bwd4::Params;

template <int D>
struct Cfg : bwd4::Cfg<D> {
  static constexpr int kBarBytes = 152 + 4 * bwd4::Cfg<D>::kLiveWords;
  static constexpr int kMaxSmem = 232448;
  static constexpr int kSmemBytes = (bwd4::Cfg<D>::kPayload + kBarBytes + 1024 <= kMaxSmem)
                                        ? bwd4::Cfg<D>::kPayload + kBarBytes + 1024
                                        : kMaxSmem;
  static constexpr int kMaxPad = kSmemBytes - bwd4::Cfg<D>::kPayload - kBarBytes;
};

template <int D, bool kGrid>
__global__ void __launch_bounds__(kThreads, 1) lao_bwd7_kernel(const __grid_constant__ Params p) {
  using C = Cfg<D>;
  static_assert(D == 128, "2-SM backward: head_dim 128");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem;
  {
    const uint32_t s = ptx::smem_u32(smem_raw);
    const uint32_t pad = (1024u - (s & 1023u)) & 1023u;
    if (pad > (uint32_t)C::kMaxPad) {   // (never on a conforming toolchain) both CTAs agree
      if (threadIdx.x == 0 && p.hop.flags) atomicOr(p.hop.flags, 4);
      return;
    }
    smem = smem_raw + pad;
  }
  uint8_t* sK = smem;
  uint8_t* sV = sK + C::kTileBytes;
  uint8_t* sQ = sV + C::kTileBytes;            // [2] stages of [QR 16 KB | QC 16 KB]
  uint8_t* sdO = sQ + 2 * C::kTileBytes;       // [dOR 16 KB | dOC 16 KB]
  uint8_t* sdS = sdO + C::kTileBytes;
  float* sStage = reinterpret_cast<float*>(sdS + C::kDsBytes);
  float* sStat = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(sStage) + 2 * C::kQuarterBytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sStat) + 2 * C::kStatBytes);
  uint64_t* kv_full = bars;          // leader: both CTAs' K/V
  uint64_t* qdo_full = bars + 1;     // [2] leader: both CTAs' Q halves + its stats; peer: its stats
  uint64_t* qdo_empty = bars + 3;    // [2] multicast: the leader's dK_i read the stage
  uint64_t* s_full = bars + 5;       // multicast
  uint64_t* p_full = bars + 6;       // leader: 2 x 256 arrivals
  uint64_t* ds_full = bars + 7;      // local: dS stored for this CTA's dQ
  uint64_t* ds_empty = bars + 8;     // local
  uint64_t* dq_full = bars + 9;      // local
  uint64_t* dq_empty = bars + 10;    // leader: 2 x 128 arrivals
  uint64_t* dkv_full = bars + 11;    // multicast
  uint64_t* dp_full = bars + 12;     // multicast
  uint64_t* do_full = bars + 13;     // leader: both CTAs' dO halves
  uint64_t* do_empty = bars + 14;    // multicast
  uint64_t* dst_full = bars + 15;    // leader: 2 x 256 arrivals (dS^T in TMEM)
  uint64_t* dk_done = bars + 16;     // multicast: dK_i done (dS^T columns free for dQ_i)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 17);

  const burst_hop& hp = p.hop;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.z, h = blockIdx.y;
  const int64_t bh = (int64_t)b * hp.heads + h;
  const int64_t k0 = hp.k_begin + (int64_t)blockIdx.x * BN;
  const int64_t k_end = hp.k_begin + hp.k_len;
  const uint32_t crank = ptx::cluster_rank();
  const bool leader = crank == 0;
  const int64_t kw0 = hp.k_begin + (int64_t)(blockIdx.x & ~1u) * BN;
  const int64_t kwrows = (kw0 + 2 * BN < k_end ? kw0 + 2 * BN : k_end) - kw0;
  const int64_t q_end = hp.q_begin + hp.q_len;
  const int64_t NTq = ceil_div(hp.n_q, 128);
  const int64_t NTk = ceil_div(hp.n_k, 128);

  int64_t qlo = hp.q_begin;
  if (hp.causal) {
    const int64_t first_q = count_le(hp.q_map, hp.n_q, pos_of(hp.k_map, kw0) - 1);
    if (first_q > qlo) qlo = first_q;
  }
  const int64_t qs = (qlo / BM) * BM;
  const int nq = qs < q_end ? (int)ceil_div(q_end - qs, BM) : 0;
  const unsigned walker = blockIdx.x >> 1;
  const int rot = nq > 0 ? (int)((walker * (unsigned)BURST_BWD_ROT) % (unsigned)nq) : 0;
  auto qtile = [&](int i) -> int64_t { int j = i + rot; if (j >= nq) j -= nq; return qs + (int64_t)j * BM; };
  auto live = [&](int i) -> bool {
    if (!kGrid) return true;
    const int64_t q0 = qtile(i) < hp.q_begin ? hp.q_begin : qtile(i);
    return grid_rect_live(hp, q0, (qtile(i) + BM < q_end ? qtile(i) + BM : q_end) - q0, kw0, kwrows);
  };
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
  int nlive = nq;

  if (warp == 12) {
    if (lane == 0) {
      ptx::mbar_init(kv_full, 1);
      for (int s = 0; s < 2; ++s) {
        ptx::mbar_init(qdo_full + s, 1);
        ptx::mbar_init(qdo_empty + s, 1);
      }
      ptx::mbar_init(s_full, 1);
      ptx::mbar_init(p_full, 4 * BN);
      ptx::mbar_init(ds_full, 2 * BN);
      ptx::mbar_init(dst_full, 4 * BN);
      ptx::mbar_init(ds_empty, 1);
      ptx::mbar_init(dq_full, 1);
      ptx::mbar_init(dq_empty, 2 * BM);
      ptx::mbar_init(dkv_full, 1);
      ptx::mbar_init(dp_full, 1);
      ptx::mbar_init(do_full, 1);
      ptx::mbar_init(do_empty, 1);
      ptx::mbar_init(dk_done, 1);
      ptx::fence_mbar_init();
      ptx::tma_prefetch_desc(&p.tm_q);
      ptx::tma_prefetch_desc(&p.tm_q64);
      ptx::tma_prefetch_desc(&p.tm_k);
      ptx::tma_prefetch_desc(&p.tm_v);
      ptx::tma_prefetch_desc(&p.tm_do);
      ptx::tma_prefetch_desc(&p.tm_do64);
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
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tbase = *tmem_holder;
  if (kGrid) nlive = (int)tmem_holder[1];
  constexpr uint32_t kS = 0, kDP = 128, kDV = 256, kDK = 256 + D;
  // shared::cluster addresses of the leader's barriers (peer bit cleared)
  const uint32_t L_kv_full = ptx::leader_addr(kv_full), L_do_full = ptx::leader_addr(do_full);
  const uint32_t L_p_full = ptx::leader_addr(p_full), L_dst_full = ptx::leader_addr(dst_full);
  const uint32_t L_dq_empty = ptx::leader_addr(dq_empty);
  constexpr int kHalf = C::kTileBytes / 2;   // 16 KB: QR / QC, dOR / dOC
  if (warp >= 12) {
   ptx::regs_dec<80>();
   if (warp == 12) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && nlive > 0) {
      // own K / V (A of the 2-SM S^T / dP^T and B of this CTA's dQ): completion on the
      // leader's barrier, which expects both CTAs' bytes
      if (leader) ptx::mbar_expect_tx(kv_full, 4 * C::kTileBytes);
      for (int x = 0; x < C::kBoxes; ++x) {
        ptx::tma_load_4d_2sm(sK + x * C::kBoxBytes, &p.tm_k, L_kv_full, x * 64, h, (int)k0, b);
        ptx::tma_load_4d_2sm(sV + x * C::kBoxBytes, &p.tm_v, L_kv_full, x * 64, h, (int)k0, b);
      }
      auto load_q = [&](int j, int ti) {
        const int s = j & 1;
        const int64_t q0 = qtile(ti);
        uint8_t* st = sQ + s * C::kTileBytes;
        ptx::mbar_wait(qdo_empty + s, ((j >> 1) & 1) ^ 1);
        ptx::mbar_expect_tx(qdo_full + s, (leader ? 2 * C::kTileBytes : 0) + C::kStatBytes);
        const uint32_t L_full = ptx::leader_addr(qdo_full + s);
        // QR: rows [64c, 64c+64) of both column boxes; QC: column box c, all rows
        ptx::tma_load_4d_2sm(st, &p.tm_q64, L_full, 0, h, (int)(q0 + 64 * crank), b);
        ptx::tma_load_4d_2sm(st + 8192, &p.tm_q64, L_full, 64, h, (int)(q0 + 64 * crank), b);
        ptx::tma_load_4d_2sm(st + kHalf, &p.tm_q, L_full, (int)crank * 64, h, (int)q0, b);
        const float* stt = p.stats + bh * NTq * 128 + q0;
        bwd4::bulk_load(sStat + s * 2 * BM, stt, BM * 4, qdo_full + s);
        bwd4::bulk_load(sStat + s * 2 * BM + BM, stt + (int64_t)hp.batch * hp.heads * NTq * 128,
                        BM * 4, qdo_full + s);
      };
      auto load_do = [&](int j, int ti) {
        const int64_t q0 = qtile(ti);
        ptx::mbar_wait(do_empty, (j & 1) ^ 1);
        if (leader) ptx::mbar_expect_tx(do_full, 2 * C::kTileBytes);
        ptx::tma_load_4d_2sm(sdO, &p.tm_do64, L_do_full, 0, h, (int)(q0 + 64 * crank), b);
        ptx::tma_load_4d_2sm(sdO + 8192, &p.tm_do64, L_do_full, 64, h, (int)(q0 + 64 * crank), b);
        ptx::tma_load_4d_2sm(sdO + kHalf, &p.tm_do, L_do_full, (int)crank * 64, h, (int)q0, b);
      };
      int tq = next_live(0), td = tq;
      load_q(0, tq); tq = next_live(tq + 1);
      load_do(0, td); td = next_live(td + 1);
      if (nlive > 1) { load_q(1, tq); tq = next_live(tq + 1); }
      for (int i = 0; i < nlive; ++i) {
        if (i + 1 < nlive) { load_do(i + 1, td); td = next_live(td + 1); }
        if (i + 2 < nlive) { load_q(i + 2, tq); tq = next_live(tq + 1); }
      }
    }
   } else if (warp == 13) {
    // ------------------------------------------------------------ MMA issue
    // Leader: the 2-SM MMAs (dV_i | S^T_{i+1} | dK_i | dP^T_{i+1}) and its own dQ_i.
    // Peer: its own dQ_i only.
    if (nlive > 0) {
      constexpr uint32_t id2_kk = ptx::make_idesc_bf16(2 * BN, BM, 0, 0);   // S^T, dP^T: M=256
      constexpr uint32_t id2_kmn = ptx::make_idesc_bf16(2 * BN, D, 0, 1);  // dV, dK: M=256, B MN
      constexpr uint32_t id_mnmn = ptx::make_idesc_bf16(BM, D, 1, 1);      // dQ (1-SM)
      const uint64_t dK = ptx::make_sdesc(ptx::smem_u32(sK), 0, 1024);
      const uint64_t dV = ptx::make_sdesc(ptx::smem_u32(sV), 0, 1024);
      const uint64_t dQR0 = ptx::make_sdesc(ptx::smem_u32(sQ), 0, 1024);          // K-major, 64 rows
      const uint64_t dQC0 = ptx::make_sdesc(ptx::smem_u32(sQ + kHalf), 0, 1024);  // MN-major, 64 cols
      const uint64_t dOR = ptx::make_sdesc(ptx::smem_u32(sdO), 0, 1024);
      const uint64_t dOC = ptx::make_sdesc(ptx::smem_u32(sdO + kHalf), 0, 1024);
      const uint64_t dSm = ptx::make_sdesc(ptx::smem_u32(sdS), 16384, 1024);
      const uint64_t dKm = ptx::make_sdesc(ptx::smem_u32(sK), C::kBoxBytes, 1024);
      constexpr uint64_t kStage = (uint64_t)(C::kTileBytes >> 4);
      auto kmaj = [](int kk) -> uint64_t { return (uint64_t)(((kk >> 2) * C::kBoxBytes + (kk & 3) * 32) >> 4); };
      auto kmaj_r = [](int kk) -> uint64_t { return (uint64_t)(((kk >> 2) * 8192 + (kk & 3) * 32) >> 4); };
      auto st_mma = [&](int stage) {   // S^T = K Q^T, M = 256 keys of the pair
        if (ptx::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            ptx::mma2_ss(tbase + kS, dK + kmaj(kk), dQR0 + stage * kStage + kmaj_r(kk), id2_kk, kk > 0);
          ptx::mma2_commit(s_full);
        }
        __syncwarp();
      };
      auto dpt_mma = [&]() {  // dP^T = V dO^T
        if (ptx::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            ptx::mma2_ss(tbase + kDP, dV + kmaj(kk), dOR + kmaj_r(kk), id2_kk, kk > 0);
          ptx::mma2_commit(dp_full);
        }
        __syncwarp();
      };
      auto dk_mma = [&](int i) {   // dK += dS^T Q (A = dS^T in each CTA's TMEM)
        if (ptx::elect_one()) {
          const uint64_t qm = dQC0 + (i & 1) * kStage;
#pragma unroll
          for (int kk = 0; kk < BM / 16; ++kk)
            ptx::mma2_ts(tbase + kDK, tbase + kDP + (kk < 4 ? kk * 8 : 32 + kk * 8),
                         qm + (uint64_t)(kk * 2048 >> 4), id2_kmn, (i > 0 || kk > 0) ? 1u : 0u);
          ptx::mma2_commit(qdo_empty + (i & 1));
          ptx::mma2_commit(dk_done);
        }
        __syncwarp();
      };
      auto dq_mma = [&]() {   // own dQ_i = dS K (1-SM) into the dP^T columns
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
      if (leader) {
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
          ptx::mbar_wait(p_full, i & 1);
          ptx::tc_fence_after();
          if (ptx::elect_one()) {   // dV += P^T dO (A = P^T in each CTA's TMEM)
#pragma unroll
            for (int kk = 0; kk < BM / 16; ++kk)
              ptx::mma2_ts(tbase + kDV, tbase + kS + (kk < 4 ? kk * 8 : 32 + kk * 8),
                           dOC + (uint64_t)(kk * 2048 >> 4), id2_kmn, (i > 0 || kk > 0) ? 1u : 0u);
            ptx::mma2_commit(do_empty);
          }
          __syncwarp();
          bool st_done = !more, dk_issued = false, dq_issued = false;
          while (!st_done || !dq_issued) {
            if (!st_done && ptx::mbar_try_wait(qdo_full + (s ^ 1), ((i + 1) >> 1) & 1)) {
              ptx::tc_fence_after();
              st_mma(s ^ 1);
              st_done = true;
            }
            if (!dk_issued && ptx::mbar_try_wait(dst_full, i & 1)) {
              ptx::tc_fence_after();
              dk_mma(i);
              dk_issued = true;
            }
            if (dk_issued && !dq_issued && ptx::mbar_try_wait(ds_full, i & 1) &&
                ptx::mbar_try_wait(dk_done, i & 1)) {
              // a 1-SM MMA is not ordered after an earlier 2-SM one on this SM: wait until
              // dK_i has read the dS^T columns dQ_i overwrites
              ptx::tc_fence_after();
              dq_mma();
              dq_issued = true;
            }
          }
          if (more) {
            ptx::mbar_wait(dq_empty, i & 1);      // both CTAs drained dQ_i
            ptx::mbar_wait(do_full, (i + 1) & 1);
            ptx::tc_fence_after();
            dpt_mma();
          }
        }
        if (ptx::elect_one()) ptx::mma2_commit(dkv_full);
        __syncwarp();
      } else {
        for (int i = 0; i < nlive; ++i) {
          ptx::mbar_wait(dk_done, i & 1);          // the leader's dK_i read this CTA's dS^T
          ptx::mbar_wait(ds_full, i & 1);
          ptx::tc_fence_after();
          dq_mma();
        }
      }
    }
   }
  } else if (warp < 8) {
    // ------------------------------------------------------------ P / dS, query half hq
    ptx::regs_inc<144>();
    const int hq = warp >> 2;
    const int t = threadIdx.x & 127;
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
      int64_t lo64 = qfirst - q0, hi64 = q_end - q0;
      const int lo = lo64 < 0 ? 0 : (lo64 > 64 ? 64 : (int)lo64);
      const int hi = !kvalid ? 0 : (hi64 > 64 ? 64 : (hi64 < 0 ? 0 : (int)hi64));
      uint64_t gq = 0;
      if (kGrid) {
        const int nv = hi64 > 64 ? 64 : (hi64 < 0 ? 0 : (int)hi64);
        if (nv > 0) gq = grid_query_bits(hp, q0, nv, kpos);
      }
      const bool warp_full = __all_sync(0xffffffffu, lo == 0 && hi == 64 && gq == 0);
      ptx::mbar_wait(qdo_full + s, (i >> 1) & 1);   // (the peer: its stats)
      ptx::mbar_wait(s_full, i & 1);
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
#pragma unroll
        for (int c4 = 0; c4 < 16; ++c4) {
          const float4 L = lse4[c4];
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
        ptx::tmem_st32(tbase + lane_off + kS + 64 * hq, pk);
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive_to(L_p_full, leader, p_full);

      ptx::mbar_wait(dp_full, i & 1);
      ptx::mbar_wait(ds_empty, (i & 1) ^ 1);
      ptx::tc_fence_after();
      uint8_t* rowp = sdS + hq * 16384 + t * 128;
      uint32_t rr[64];
      ptx::tmem_ld32(tbase + lane_off + kDP + 64 * hq, *reinterpret_cast<uint32_t(*)[32]>(rr));
      ptx::tmem_ld32(tbase + lane_off + kDP + 64 * hq + 32, *reinterpret_cast<uint32_t(*)[32]>(rr + 32));
      ptx::tmem_wait_ld();
      ptx::reg_fence(rr);
      uint32_t pks[32];
#pragma unroll
      for (int qc = 0; qc < 2; ++qc) {
        const uint32_t* r = rr + 32 * qc;
        uint32_t* pk = pks + 16 * qc;
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          const float4 Dv = dst4[qc * 8 + j4];
          const int c = qc * 32 + 4 * j4;
          const float2 da = ptx::fmul2(make_float2(pr[c], pr[c + 1]),
                                       ptx::fadd2(make_float2(__uint_as_float(r[4 * j4]), __uint_as_float(r[4 * j4 + 1])),
                                                  make_float2(-Dv.x, -Dv.y)));
          const float2 db = ptx::fmul2(make_float2(pr[c + 2], pr[c + 3]),
                                       ptx::fadd2(make_float2(__uint_as_float(r[4 * j4 + 2]), __uint_as_float(r[4 * j4 + 3])),
                                                  make_float2(-Dv.z, -Dv.w)));
          pk[2 * j4] = ptx::pack_bf16(da.x, da.y);
          pk[2 * j4 + 1] = ptx::pack_bf16(db.x, db.y);
        }
        ptx::tmem_st16(tbase + lane_off + kDP + 64 * hq + 16 * qc,
                       *reinterpret_cast<const uint32_t(*)[16]>(pk));
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive_to(L_dst_full, leader, dst_full);
#pragma unroll
      for (int qc = 0; qc < 2; ++qc) {
        const uint32_t* pk = pks + 16 * qc;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int ch = qc * 4 + u;
          *reinterpret_cast<uint4*>(rowp + ((ch ^ (t & 7)) << 4)) =
              make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
      }
      ptx::fence_proxy_async_smem();
      ptx::tc_fence_before();
      ptx::mbar_arrive(ds_full);
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
    ptx::regs_inc<144>();
    const int t = threadIdx.x & 127;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    float4* stg = reinterpret_cast<float4*>(sStage);
    for (int i = 0, ti = next_live(0); i < nlive; ++i, ti = next_live(ti + 1)) {
      const int64_t q0 = qtile(ti);
      const bool qvalid = q0 + t >= hp.q_begin && q0 + t < q_end && q0 + t < hp.n_q;
      ptx::mbar_wait(dq_full, i & 1);
      ptx::tc_fence_after();
      uint32_t r[D];
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc)
        ptx::tmem_ld32(tbase + lane_off + kDP + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(r + cc * 32));
      ptx::tmem_wait_ld();
      ptx::reg_fence(r);
      ptx::tc_fence_before();
      ptx::mbar_arrive_to(L_dq_empty, leader, dq_empty);
      const float sc = qvalid ? p.scale : 0.f;
#pragma unroll
      for (int qq = 0; qq < D / 32; ++qq) {
        float4* buf = stg + (qq & 1) * (8 * 128);
        if (t == 0) ptx::bulk_wait_read<1>();
        ptx::named_bar_sync(1, 128);
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
    }
    if (t == 0) ptx::bulk_wait_all();
  }

  __syncwarp();
  ptx::tc_fence_before();
  ptx::cluster_sync();   // no 2-SM MMA, load or remote arrive may target an exited CTA
  if (warp == 12) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tbase, 512);
  }
}

}  // namespace bwd7
}  // namespace burst
