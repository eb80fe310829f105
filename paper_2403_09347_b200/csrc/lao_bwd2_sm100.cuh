// LAO backward on sm_100a with CTA PAIRS (cta_group::2), head_dim 128.
//
// Same math as lao_bwd_sm100.cuh (local_backward, local_attn.py:255-353), but a
// pair of CTAs (one cluster) owns 256 keys, so every dQ partial written to the
// fp32 workspace already sums over 256 keys: half the L2 reduction volume of the
// single-CTA kernel, whose ceiling that volume sets (~3.5 TB/s of fp32 reduction,
// profiles/r01_reduction_microbench.txt).
//
// CTA c of the pair owns keys [k0 + 128c, +128).  All MMAs are issued by the
// leader (c = 0) with cta_group::2 and both SMs' tensor cores:
//   S^T  = K Q^T   M=256 keys, N=128 queries (B = query half c of Q per CTA)
//   dP^T = V dO^T  (same shape)
//   dV  += P^T dO  M=256 keys, N=128 d (B = d half c of dO), A = P^T in TMEM
//   dK  += dS^T Q  (same shape), A = dS^T in TMEM
//   dQ   = dS K    M=128 queries (64 per CTA), N=128 d, K=256 keys: A = dS for this
//                  CTA's 64 queries over BOTH CTAs' keys (the peer's half arrives
//                  through DSMEM), B = K[256 keys][d half c]
// TMEM per CTA: [0,128) S^T -> P^T(bf16, cols 0-63);  [128,256) dP^T -> dQ (cols
// 128-191, "2x2" layout: lane = query%64 + 64*(d/64), col = d%64) and dS^T (bf16,
// cols 192-255); [256,384) dV; [384,512) dK.
// SMEM per CTA (~196 KB): K, V, K_dQ, dS_dQ (32 KB each), and one 16 KB buffer per
// operand slab Qa = Q[64 q of half c][128 d], Qb = Q[128 q][64 d of half c], dOa, dOb,
// each reloaded as soon as the MMA that read it retires (a full iteration of slack).
// Warps: 0-3 P/dS (thread = own key row), 4-7 dQ drain (thread = TMEM lane),
// 8 TMA producer + TMEM allocator, 9 MMA issuer (leader only), 10-11 idle.
#pragma once
#include <cuda.h>
#include "common.cuh"
#include "ptx.cuh"

namespace burst {
namespace bwd2 {

constexpr int D = 128;
constexpr int BM = 128;          // queries per iteration
constexpr int BN = 128;          // keys per CTA (256 per pair)
constexpr int kThreads = 384;
constexpr int kStatSlots = 3;

struct Params {
  CUtensorMap tm_q128, tm_q64, tm_do128, tm_do64, tm_k, tm_v;
  const float* stats;   // [2][B*H][NTq*128]: lse*log2e, D
  float* dq_acc;        // TL over n_q
  float* dk_acc;        // TL over n_k
  float* dv_acc;
  burst_hop hop;
  float scale_log2, scale;
  int accumulate;
  long long* trace;   // BURST_TRACE builds only
};

namespace L {   // shared-memory layout (bytes from the 1024-aligned base)
constexpr int K = 0, V = 32768, KQ = 65536, DSQ = 98304;
constexpr int QA = 131072, QB = 147456, DOA = 163840, DOB = 180224;
constexpr int XS = 196608;                       // outgoing dS half for the peer (16 KB)
constexpr int STATS = 212992;                    // kStatSlots x (lse2[128], D[128])
constexpr int BARS = STATS + kStatSlots * 1024;  // barriers
constexpr int kBytes = BARS + 64 * 8;
}  // namespace L
constexpr int kSmemBytes = L::kBytes + 1024;

// barrier indices
enum {
  B_KV = 0, B_QA_F, B_QA_E, B_QB_F, B_QB_E, B_DA_F, B_DA_E, B_DB_F, B_DB_E,
  B_ST_F, B_ST_E = B_ST_F + kStatSlots,
  B_S = B_ST_E + kStatSlots, B_DP, B_P, B_DS, B_DQF, B_DQE, B_DSQE, B_DKV, B_X, B_XR, B_COUNT
};

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          ptx::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(ptx::smem_u32(bar))
      : "memory");
}

#ifdef BURST_TRACE
#define BTRACE2(ev, i)                                                                       \
  do {                                                                                       \
    if (p.trace && blockIdx.x < 2 && blockIdx.y == 0 && blockIdx.z == 0 && (i) < 64)         \
      p.trace[(blockIdx.x * 16 + (ev)) * 64 + (i)] = clock64();                              \
  } while (0)
#else
#define BTRACE2(ev, i)
#endif

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    lao_bwd2_kernel(const __grid_constant__ Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm;
  {
    const uint32_t s = ptx::smem_u32(smem_raw);
    sm = smem_raw + ((1024u - (s & 1023u)) & 1023u);
  }
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BARS);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bar + B_COUNT);
  float* sStat = reinterpret_cast<float*>(sm + L::STATS);

  const burst_hop& hp = p.hop;
  const uint32_t crank = ptx::cluster_rank();
  const bool leader = crank == 0;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.z, h = blockIdx.y;
  const int64_t bh = (int64_t)b * hp.heads + h;
  const int64_t kpair = hp.k_begin + (int64_t)(blockIdx.x >> 1) * (2 * BN);
  const int64_t k0 = kpair + (int64_t)crank * BN;            // this CTA's first key
  const int64_t k_end = hp.k_begin + hp.k_len;
  const int64_t q_end = hp.q_begin + hp.q_len;
  const int64_t NTq = ceil_div(hp.n_q, 128);
  const int64_t NTk = ceil_div(hp.n_k, 128);

  // Query tiles: both CTAs must walk the same sequence (shared MMAs); causal =>
  // the suffix visible to the pair's first key.
  int64_t qs = hp.q_begin;
  if (hp.causal) {
    const int64_t first_q = count_le(hp.q_map, hp.n_q, pos_of(hp.k_map, kpair) - 1);
    if (first_q > qs) qs = hp.q_begin + ((first_q - hp.q_begin) / BM) * BM;
  }
  const int nq = qs < q_end ? (int)ceil_div(q_end - qs, BM) : 0;
  const int rot = nq > 0 ? (int)(((blockIdx.x >> 1) * 7u) % (unsigned)nq) : 0;
  auto qtile = [&](int i) -> int64_t {
    int j = i + rot;
    if (j >= nq) j -= nq;
    return qs + (int64_t)j * BM;
  };

  if (warp == 8) {
    if (lane == 0) {
      for (int i = 0; i < B_COUNT; ++i) {
        uint32_t cnt = 1;
        if (i >= B_ST_E && i < B_ST_E + kStatSlots) cnt = BN;
        if (i == B_P || i == B_DS || i == B_DQE) cnt = 2 * BN;   // both CTAs arrive
        ptx::mbar_init(bar + i, cnt);
      }
      ptx::fence_mbar_init();
    }
    __syncwarp();
    ptx::tmem_alloc_2sm(tmem_holder, 512);
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tbase = *tmem_holder;
  constexpr uint32_t kS = 0, kDP = 128, kDQ = 128, kDST = 192, kDV = 256, kDK = 384;

  if (warp >= 8) {
    ptx::regs_dec<88>();
    if (warp == 8 && lane == 0 && nq > 0) {
      // ------------------------------------------------------------ TMA producer
      const int qd = (int)crank * 64;          // this CTA's d half (Qb, dOb, K_dQ)
      auto full = [&](int id) { return ptx::leader_addr(bar + id); };
      auto arm = [&](int id, uint32_t bytes) {   // leader posts both CTAs' bytes
        if (leader) ptx::mbar_expect_tx(bar + id, 2 * bytes);
      };
      arm(B_KV, 3 * 32768);
      for (int x = 0; x < 2; ++x) {
        ptx::tma_load_4d_2sm(sm + L::K + x * 16384, &p.tm_k, full(B_KV), x * 64, h, (int)k0, b);
        ptx::tma_load_4d_2sm(sm + L::V + x * 16384, &p.tm_v, full(B_KV), x * 64, h, (int)k0, b);
        ptx::tma_load_4d_2sm(sm + L::KQ + x * 16384, &p.tm_k, full(B_KV), qd, h,
                             (int)(kpair + x * BN), b);
      }
      int nqa = 0, nqb = 0, nda = 0, ndb = 0, nst = 0;
      auto load_qa = [&](int i) {
        ptx::mbar_wait(bar + B_QA_E, (nqa & 1) ^ 1);
        ++nqa;
        arm(B_QA_F, 16384);
        const int r = (int)(qtile(i) + crank * 64);
        ptx::tma_load_4d_2sm(sm + L::QA, &p.tm_q64, full(B_QA_F), 0, h, r, b);
        ptx::tma_load_4d_2sm(sm + L::QA + 8192, &p.tm_q64, full(B_QA_F), 64, h, r, b);
      };
      auto load_da = [&](int i) {
        ptx::mbar_wait(bar + B_DA_E, (nda & 1) ^ 1);
        ++nda;
        arm(B_DA_F, 16384);
        const int r = (int)(qtile(i) + crank * 64);
        ptx::tma_load_4d_2sm(sm + L::DOA, &p.tm_do64, full(B_DA_F), 0, h, r, b);
        ptx::tma_load_4d_2sm(sm + L::DOA + 8192, &p.tm_do64, full(B_DA_F), 64, h, r, b);
      };
      auto load_qb = [&](int i) {
        ptx::mbar_wait(bar + B_QB_E, (nqb & 1) ^ 1);
        ++nqb;
        arm(B_QB_F, 16384);
        ptx::tma_load_4d_2sm(sm + L::QB, &p.tm_q128, full(B_QB_F), qd, h, (int)qtile(i), b);
      };
      auto load_db = [&](int i) {
        ptx::mbar_wait(bar + B_DB_E, (ndb & 1) ^ 1);
        ++ndb;
        arm(B_DB_F, 16384);
        ptx::tma_load_4d_2sm(sm + L::DOB, &p.tm_do128, full(B_DB_F), qd, h, (int)qtile(i), b);
      };
      auto load_st = [&](int i) {     // local: each CTA needs all 128 queries' stats
        const int s = nst % kStatSlots;
        ptx::mbar_wait(bar + B_ST_E + s, ((nst / kStatSlots) & 1) ^ 1);
        ++nst;
        ptx::mbar_expect_tx(bar + B_ST_F + s, 1024);
        const float* st = p.stats + bh * NTq * 128 + qtile(i);
        bulk_load(sStat + s * 256, st, 512, bar + B_ST_F + s);
        bulk_load(sStat + s * 256 + 128, st + (int64_t)hp.batch * hp.heads * NTq * 128, 512,
                  bar + B_ST_F + s);
      };
      // release order of the single buffers (see the MMA issuer) drives the load order
      load_st(0); load_qa(0); load_da(0); load_qb(0); load_db(0);
      if (nq > 1) { load_st(1); load_qa(1); load_da(1); }
      for (int i = 0; i < nq; ++i) {
        if (i + 1 < nq) load_db(i + 1);
        if (i + 2 < nq) { load_st(i + 2); load_qa(i + 2); }
        if (i + 1 < nq) load_qb(i + 1);
        if (i + 2 < nq) load_da(i + 2);
      }
    } else if (warp == 9 && lane == 0 && leader && nq > 0) {
      // ------------------------------------------------------------ MMA issuer (leader)
      constexpr uint32_t id_st = ptx::make_idesc_bf16(256, BM, 0, 0);   // S^T, dP^T
      constexpr uint32_t id_kd = ptx::make_idesc_bf16(256, D, 0, 1);    // dV, dK
      constexpr uint32_t id_dq = ptx::make_idesc_bf16(128, D, 1, 1);    // dQ (64 rows / CTA)
      const uint32_t a0 = ptx::smem_u32(sm);
      auto kmajor = [&](uint32_t base, int kk, uint32_t box_bytes) {
        return ptx::make_sdesc(base + (kk >> 2) * box_bytes + (kk & 3) * 32, 0, 1024);
      };
      ptx::mbar_wait(bar + B_KV, 0);
      auto st_mma = [&]() {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          ptx::mma2_ss(tbase + kS, kmajor(a0 + L::K, kk, 16384), kmajor(a0 + L::QA, kk, 8192),
                       id_st, kk > 0);
      };
      auto dpt_mma = [&]() {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          ptx::mma2_ss(tbase + kDP, kmajor(a0 + L::V, kk, 16384), kmajor(a0 + L::DOA, kk, 8192),
                       id_st, kk > 0);
      };
      ptx::mbar_wait(bar + B_QA_F, 0);
      ptx::tc_fence_after();
      st_mma();
      ptx::mma2_commit(bar + B_S);
      ptx::mma2_commit(bar + B_QA_E);
      ptx::mbar_wait(bar + B_DA_F, 0);
      ptx::tc_fence_after();
      dpt_mma();
      ptx::mma2_commit(bar + B_DP);
      ptx::mma2_commit(bar + B_DA_E);
      for (int i = 0; i < nq; ++i) {
        const bool more = i + 1 < nq;
        // dV += P^T dO
        ptx::mbar_wait(bar + B_P, i & 1); BTRACE2(0, i);
        ptx::mbar_wait(bar + B_DB_F, i & 1); BTRACE2(9, i);
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BM / 16; ++kk)
          ptx::mma2_ts(tbase + kDV, tbase + kS + kk * 8,
                       ptx::make_sdesc(a0 + L::DOB + kk * 2048, 0, 1024), id_kd,
                       (i > 0 || kk > 0) ? 1u : 0u);
        ptx::mma2_commit(bar + B_DB_E);
        if (more) {   // S^T_{i+1} overlaps the dS_i phase
          ptx::mbar_wait(bar + B_QA_F, (i + 1) & 1); BTRACE2(11, i);
          ptx::tc_fence_after();
          st_mma();
          ptx::mma2_commit(bar + B_S);
          ptx::mma2_commit(bar + B_QA_E);
        }
        // dK += dS^T Q ; dQ = dS K
        ptx::mbar_wait(bar + B_DS, i & 1); BTRACE2(1, i);
        ptx::mbar_wait(bar + B_QB_F, i & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BM / 16; ++kk)
          ptx::mma2_ts(tbase + kDK, tbase + kDST + kk * 8,
                       ptx::make_sdesc(a0 + L::QB + kk * 2048, 0, 1024), id_kd,
                       (i > 0 || kk > 0) ? 1u : 0u);
        ptx::mma2_commit(bar + B_QB_E);
        ptx::mbar_wait(bar + B_X, i & 1);     // peer's dS half landed here
        ptx::mbar_wait(bar + B_XR, i & 1);    // ... and ours landed in the peer (relayed)
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < (2 * BN) / 16; ++kk)
          ptx::mma2_ss(tbase + kDQ, ptx::make_sdesc(a0 + L::DSQ + kk * 2048, 0, 1024),
                       ptx::make_sdesc(a0 + L::KQ + kk * 2048, 0, 1024), id_dq, kk > 0);
        ptx::mma2_commit(bar + B_DQF);
        ptx::mma2_commit(bar + B_DSQE);
        if (more) {
          ptx::mbar_wait(bar + B_DQE, i & 1); BTRACE2(2, i);
          ptx::mbar_wait(bar + B_DA_F, (i + 1) & 1); BTRACE2(10, i);
          ptx::tc_fence_after();
          dpt_mma();
          ptx::mma2_commit(bar + B_DP);
          ptx::mma2_commit(bar + B_DA_E);
        }
      }
      ptx::mma2_commit(bar + B_DKV);
    } else if (warp == 10 && lane == 0 && !leader && nq > 0) {
      // relay: tell the leader that the leader's dS half has landed in this CTA
      const uint32_t xr = ptx::leader_addr(bar + B_XR);
      for (int i = 0; i < nq; ++i) {
        ptx::mbar_wait(bar + B_X, i & 1);
        ptx::mbar_arrive_remote(xr);
      }
    }
  } else if (warp < 4) {
    // ------------------------------------------------------------ P / dS warpgroup
    ptx::regs_inc<240>();
    const int t = threadIdx.x;                 // own key row = TMEM lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int64_t krow = k0 + t;
    const bool kvalid = krow < k_end && krow < hp.n_k;
    const int64_t kpos = (hp.causal || hp.grid_skip) ? pos_of(hp.k_map, kvalid ? krow : k0) : 0;
    const int64_t qfirst = hp.causal ? count_le(hp.q_map, hp.n_q, kpos - 1) : 0;
    const float c2 = p.scale_log2;
    const uint32_t p_bar = ptx::leader_addr(bar + B_P), ds_bar = ptx::leader_addr(bar + B_DS);
    const uint32_t xs_peer = ptx::peer_addr(sm + L::DSQ + crank * 16384, crank ^ 1u);
    const uint32_t xbar_peer = ptx::peer_addr(bar + B_X, crank ^ 1u);
    uint8_t* xs_row = sm + L::XS + t * 128;
    // this key row inside both CTAs' dS_dQ buffers: row 128*crank + t (K-dim = pair's keys)
    const uint32_t dsq_row = (uint32_t)(crank * BN + t);
    uint8_t* dsq_local = sm + L::DSQ + (dsq_row >> 7) * 16384 + (dsq_row & 127) * 128;
    for (int i = 0; i < nq; ++i) {
      const int s = i % kStatSlots;
      const int64_t q0 = qtile(i);
      int64_t lo64 = qfirst - q0, hi64 = q_end - q0;
      const int lo = lo64 < 0 ? 0 : (lo64 > BM ? BM : (int)lo64);
      const int hi = !kvalid ? 0 : (hi64 > BM ? BM : (hi64 < 0 ? 0 : (int)hi64));
      uint64_t gq0 = 0, gq1 = 0;   // block-sparse grid: hidden query columns
      if (hp.grid_skip) {
        const int nv = hi64 > BM ? BM : (hi64 < 0 ? 0 : (int)hi64);
        if (nv > 0) gq0 = grid_query_bits(hp, q0, nv < 64 ? nv : 64, kpos);
        if (nv > 64) gq1 = grid_query_bits(hp, q0 + 64, nv - 64, kpos);
      }
      const bool warp_full = __all_sync(0xffffffffu, lo == 0 && hi == BM && (gq0 | gq1) == 0);
      ptx::mbar_wait(bar + B_ST_F + s, (i / kStatSlots) & 1);
      ptx::mbar_wait(bar + B_S, i & 1); BTRACE2(3, i);
      ptx::tc_fence_after();
      const float4* lse4 = reinterpret_cast<const float4*>(sStat + s * 256);
      const float4* dst4 = lse4 + BM / 4;
      float pr[BM];
      {
        uint32_t r[BM];
#pragma unroll
        for (int cc = 0; cc < BM / 32; ++cc)
          ptx::tmem_ld32(tbase + lane_off + kS + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(r + cc * 32));
        ptx::tmem_wait_ld();
        ptx::reg_fence(r);
#pragma unroll
        for (int c4 = 0; c4 < BM / 4; ++c4) {
          const float4 Lv = lse4[c4];
          pr[4 * c4 + 0] = ptx::ex2(fmaf(__uint_as_float(r[4 * c4 + 0]), c2, -Lv.x));
          pr[4 * c4 + 1] = ptx::ex2(fmaf(__uint_as_float(r[4 * c4 + 1]), c2, -Lv.y));
          pr[4 * c4 + 2] = ptx::ex2(fmaf(__uint_as_float(r[4 * c4 + 2]), c2, -Lv.z));
          pr[4 * c4 + 3] = ptx::ex2(fmaf(__uint_as_float(r[4 * c4 + 3]), c2, -Lv.w));
        }
      }
      if (!warp_full) {
#pragma unroll
        for (int c = 0; c < BM; ++c)
          if (c < lo || c >= hi || (((c < 64 ? gq0 : gq1) >> (c & 63)) & 1)) pr[c] = 0.f;
      }
#pragma unroll
      for (int cc = 0; cc < BM / 64; ++cc) {
        uint32_t pk[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) pk[j] = ptx::pack_bf16(pr[cc * 64 + 2 * j], pr[cc * 64 + 2 * j + 1]);
        ptx::tmem_st32(tbase + lane_off + kS + cc * 32, pk);
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive_to(p_bar, leader, bar + B_P); BTRACE2(4, i);

      // dS = P (dP - D); chunks of 32 queries from the top so every dS^T column
      // written into [192,256) has already been read as dP^T
      ptx::mbar_wait(bar + B_DP, i & 1); BTRACE2(5, i);
      ptx::mbar_wait(bar + B_DSQE, (i & 1) ^ 1);
      if (t == 0) ptx::mbar_expect_tx(bar + B_X, 16384);   // the peer's half of this tile
      ptx::tc_fence_after();
#pragma unroll
      for (int cc = 3; cc >= 0; --cc) {
        uint32_t r[32];
        ptx::tmem_ld32(tbase + lane_off + kDP + cc * 32, r);
        ptx::tmem_wait_ld();
        ptx::reg_fence(r);
        uint32_t pk[16];
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          const float4 Dv = dst4[cc * 8 + j4];
          const int c = cc * 32 + 4 * j4;
          pk[2 * j4] = ptx::pack_bf16(pr[c] * (__uint_as_float(r[4 * j4]) - Dv.x),
                                      pr[c + 1] * (__uint_as_float(r[4 * j4 + 1]) - Dv.y));
          pk[2 * j4 + 1] = ptx::pack_bf16(pr[c + 2] * (__uint_as_float(r[4 * j4 + 2]) - Dv.z),
                                          pr[c + 3] * (__uint_as_float(r[4 * j4 + 3]) - Dv.w));
        }
        ptx::tmem_st16(tbase + lane_off + kDST + cc * 16, pk);
        // dS_dQ (MN-major, 64 queries of one half per 128 B row): half cc/2 lives in CTA cc/2
        const int half = cc >> 1;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int ch = (cc & 1) * 4 + u;
          const uint32_t off = (uint32_t)((ch ^ (dsq_row & 7)) << 4);
          const uint4 v = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
          *reinterpret_cast<uint4*>((half == (int)crank ? dsq_local : xs_row) + off) = v;
        }
      }
      ptx::tmem_wait_st();
      ptx::fence_proxy_async_smem();
      ptx::named_bar_sync(2, BN);
      if (t == 0)   // one TMA bulk copy ships the peer's half: SMEM -> peer SMEM, tx on its B_X
        ptx::bulk_copy_to_peer(xs_peer, sm + L::XS, 16384, xbar_peer);
      ptx::tc_fence_before();
      ptx::mbar_arrive_to(ds_bar, leader, bar + B_DS); BTRACE2(6, i);
      ptx::mbar_arrive(bar + B_ST_E + s);
    }
    // -------------------------------------------------------- dK / dV epilogue
    if (nq > 0) {
      ptx::mbar_wait(bar + B_DKV, 0);
      ptx::tc_fence_after();
    }
#pragma unroll 1
    for (int which = 0; which < 2; ++which) {
      float* dst = which == 0 ? p.dv_acc : p.dk_acc;
      const float mul = which == 0 ? 1.f : p.scale;
      const uint32_t col0 = which == 0 ? kDV : kDK;
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t r[32];
        if (nq > 0) {
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
  } else if (warp < 8) {
    // ------------------------------------------------------------ dQ drain warpgroup
    // TMEM lane L holds query 64*crank + L%64, d columns 64*(L/64) + [0,64).
    const int L = threadIdx.x & 127;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int dbase = (L >> 6) * 64;
    const uint32_t dqe_bar = ptx::leader_addr(bar + B_DQE);
    for (int i = 0; i < nq; ++i) {
      const int64_t qrow = qtile(i) + crank * 64 + (L & 63);
      const bool qvalid = qrow < q_end && qrow < hp.n_q;
      ptx::mbar_wait(bar + B_DQF, i & 1); BTRACE2(7, i);
      ptx::tc_fence_after();
      uint32_t r[64];
      ptx::tmem_ld32(tbase + lane_off + kDQ, *reinterpret_cast<uint32_t(*)[32]>(r));
      ptx::tmem_ld32(tbase + lane_off + kDQ + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
      ptx::tmem_wait_ld();
      ptx::reg_fence(r);
      ptx::tc_fence_before();
      ptx::mbar_arrive_to(dqe_bar, leader, bar + B_DQE); BTRACE2(8, i);
      if (qvalid) {
        float* base = p.dq_acc + tl_index(bh, qrow, dbase, D, NTq);
#pragma unroll
        for (int j = 0; j < 64; j += 4)   // next 4-column group: 128 rows x 4 floats further
          ptx::red_add_v4(base + (size_t)(j >> 2) * 512, __uint_as_float(r[j]) * p.scale,
                          __uint_as_float(r[j + 1]) * p.scale, __uint_as_float(r[j + 2]) * p.scale,
                          __uint_as_float(r[j + 3]) * p.scale);
      }
    }
  }

  __syncwarp();
  ptx::tc_fence_before();
  ptx::cluster_sync();      // the peer may still write our dS_dQ / arrive on our barriers
  if (warp == 8) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_2sm(tbase, 512);
  }
}

}  // namespace bwd2
}  // namespace burst
