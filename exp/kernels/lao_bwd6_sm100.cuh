// LAO backward on sm_100a with CTA PAIRS, scheduled so the dS exchange and the
// dQ MMA/drain are OFF the critical path (lao_bwd5 with a different TMEM plan).
//
// In lao_bwd5 the dQ tile lives in the dP^T columns, so dP^T_{i+1} waits for
// dS_i -> DSMEM exchange (~1000 cycles) -> dQ_i -> drain: a ~4800-cycle chain per
// step (profiles/r01_trace_bwd5_c2.txt).  Here dQ_i goes to S^T columns [64,128),
// free once both P/dS warpgroups have loaded S^T_{i+1} into registers (barrier
// B_SREAD), while P^T_i packs into [0,64).  dP^T_{i+1} follows dK_i directly, and
// S^T_{i+2} only waits for dQ_i to be drained, which has most of a step of slack.
// Critical path per step: the P/dS warpgroups (exp + dS), i.e. ~2700 cycles.
//
// Same math as lao_bwd4 (local_backward, local_attn.py:255-353; ring.backward_step
// ring.py:221-242).  MMAs (leader, cta_group::2; CTA c owns keys [kp + 128c, +128)):
//   S^T  = K Q^T    M=256 keys, N=128 queries (B: Q rows [64c, 64c+64) per CTA)
//   dP^T = V dO^T   (same shape)
//   dV  += P^T dO   A = P^T in TMEM [0,64) (B: dO d-half c)
//   dK  += dS^T Q   A = dS^T in TMEM [128,192) (B: Q d-half c)
//   dQ   = dS K     M=128 queries (query half c per CTA), K = the pair's 256 keys;
//                   the peer's dS half arrives by a TMA bulk SMEM->peer copy
// TMEM per CTA: S^T [0,128) -> P^T [0,64) + dQ [64,128) ("2x2": lane = query%64 +
// 64*(d/64), col = d%64); dP^T [128,256) -> dS^T [128,192); dV [256,384); dK [384,512).
// Per step i the MMA issuer runs: dV_i | S^T_{i+1} (after dQ_{i-1} drained) | dK_i |
// dP^T_{i+1} | dQ_i (after the exchange and B_SREAD of S^T_{i+1}).
// Warps: 0-3 P/dS query half 0, 4-7 query half 1 (thread = own key row); 8-11 dQ
// drain; 12 TMA producer (+ TMEM alloc); 13 MMA issuer (leader); 14 relay (peer).
#pragma once
#include <cuda.h>
#include "common.cuh"
#include "ptx.cuh"

namespace burst {
namespace bwd6 {

constexpr int D = 128;
constexpr int BM = 128;          // queries per iteration
constexpr int BN = 128;          // keys per CTA (256 per pair)
constexpr int kThreads = 512;
constexpr int kStatSlots = 2;

struct Params {
  CUtensorMap tm_q128, tm_q64, tm_do128, tm_do64, tm_k, tm_v;
  CUtensorMap tm_dq;    // dq_acc TL viewed as f32 [groups][128 rows][4], box {4, 64, 8}
  const float* stats;   // [2][B*H][NTq*128]: lse*log2e, D
  float* dq_acc;        // TL over n_q
  float* dk_acc;        // TL over n_k
  float* dv_acc;
  burst_hop hop;
  float scale_log2, scale;
  int accumulate;
  long long* trace;     // BURST_TRACE builds only
};

namespace L {   // shared-memory layout (bytes from the 1024-aligned base)
constexpr int K = 0, V = 32768, KQ = 65536, DSQ = 98304;
constexpr int QA = 131072, QB = 147456, DOA = 163840, DOB = 180224;
constexpr int XS = 196608;                        // outgoing dS half for the peer (16 KB)
constexpr int STAGE = 212992;                     // dQ staging: 8 column groups x 64 rows (8 KB)
constexpr int STATS = STAGE + 8192;               // kStatSlots x (lse2[128], D[128])
constexpr int BARS = STATS + kStatSlots * 1024;
constexpr int kBytes = BARS + 64 * 8;
}  // namespace L
constexpr int kSmemBytes = L::kBytes + 1024;
static_assert(kSmemBytes <= 232448, "bwd6 shared memory");

enum {
  B_KV = 0, B_QA_F, B_QA_E, B_QB_F, B_QB_E, B_DA_F, B_DA_E, B_DB_F, B_DB_E,
  B_ST_F, B_ST_E = B_ST_F + kStatSlots,
  B_S = B_ST_E + kStatSlots, B_DP, B_P, B_DS, B_DQF, B_DQE, B_DSQE, B_DKV, B_X, B_XR, B_SREAD,
  B_COUNT
};

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          ptx::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(ptx::smem_u32(bar))
      : "memory");
}

#ifdef BURST_TRACE
#define BTRACE6(ev, i)                                                                       \
  do {                                                                                       \
    if (p.trace && blockIdx.x < 2 && blockIdx.y == 0 && blockIdx.z == 0 && (i) < 64)         \
      p.trace[(blockIdx.x * 16 + (ev)) * 64 + (i)] = clock64();                              \
  } while (0)
#else
#define BTRACE6(ev, i)
#endif

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    lao_bwd6_kernel(const __grid_constant__ Params p) {
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

  // both CTAs walk the same query tiles (shared MMAs); causal => the suffix
  // visible to the pair's first key
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

  if (warp == 12) {
    if (lane == 0) {
      for (int i = 0; i < B_COUNT; ++i) {
        uint32_t cnt = 1;
        if (i >= B_ST_E && i < B_ST_E + kStatSlots) cnt = 2 * BN;   // both P/dS warpgroups
        if (i == B_P || i == B_DS || i == B_SREAD) cnt = 4 * BN;     // both WGs of both CTAs
        if (i == B_DQE) cnt = 2 * BN;                                // drain WGs of both CTAs
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
  constexpr uint32_t kS = 0, kDQ = 64, kDP = 128, kDST = 128, kDV = 256, kDK = 384;

  if (warp >= 12) {
    ptx::regs_dec<112>();
    if (warp == 12 && lane == 0 && nq > 0) {
      // ------------------------------------------------------------ TMA producer
      const int qd = (int)crank * 64;          // this CTA's d half (QB, dOB, KQ)
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
      // issue order follows the order the MMA issuer releases the single buffers
      load_st(0); load_qa(0); load_da(0); load_qb(0); load_db(0);
      if (nq > 1) { load_st(1); load_qa(1); load_da(1); }
      for (int i = 0; i < nq; ++i) {
        if (i + 1 < nq) load_db(i + 1);
        if (i + 2 < nq) { load_st(i + 2); load_qa(i + 2); }
        if (i + 1 < nq) load_qb(i + 1);
        if (i + 2 < nq) load_da(i + 2);
      }
    } else if (warp == 13 && leader && nq > 0) {
      // ------------------------------------------------------------ MMA issuer (leader)
      // The whole warp runs this loop (warp-uniform control flow, so descriptors stay
      // in uniform registers); one elected lane issues each MMA group and its commits.
      // Descriptors: base computed once, + (byte offset >> 4) per K step.
      constexpr uint32_t id_st = ptx::make_idesc_bf16(256, BM, 0, 0);   // S^T, dP^T
      constexpr uint32_t id_kd = ptx::make_idesc_bf16(256, D, 0, 1);    // dV, dK
      constexpr uint32_t id_dq = ptx::make_idesc_bf16(128, D, 1, 1);    // dQ (64 rows / CTA)
      const uint32_t a0 = ptx::smem_u32(sm);
      const uint64_t dK = ptx::make_sdesc(a0 + L::K, 0, 1024), dV = ptx::make_sdesc(a0 + L::V, 0, 1024);
      const uint64_t dQA = ptx::make_sdesc(a0 + L::QA, 0, 1024), dDOA = ptx::make_sdesc(a0 + L::DOA, 0, 1024);
      const uint64_t dQB = ptx::make_sdesc(a0 + L::QB, 0, 1024), dDOB = ptx::make_sdesc(a0 + L::DOB, 0, 1024);
      const uint64_t dDSQ = ptx::make_sdesc(a0 + L::DSQ, 0, 1024), dKQ = ptx::make_sdesc(a0 + L::KQ, 0, 1024);
      auto kmaj = [](int kk, uint32_t box_bytes) -> uint64_t {   // K-major step offset >> 4
        return (uint64_t)(((kk >> 2) * box_bytes + (kk & 3) * 32) >> 4);
      };
      auto st_mma = [&]() {
        if (ptx::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            ptx::mma2_ss(tbase + kS, dK + kmaj(kk, 16384), dQA + kmaj(kk, 8192), id_st, kk > 0);
          ptx::mma2_commit(bar + B_S);
          ptx::mma2_commit(bar + B_QA_E);
        }
        __syncwarp();
      };
      auto dpt_mma = [&]() {
        if (ptx::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            ptx::mma2_ss(tbase + kDP, dV + kmaj(kk, 16384), dDOA + kmaj(kk, 8192), id_st, kk > 0);
          ptx::mma2_commit(bar + B_DP);
          ptx::mma2_commit(bar + B_DA_E);
        }
        __syncwarp();
      };
      auto dk_mma = [&](int i) {   // dK += dS^T Q (A = dS^T in TMEM [128,192))
        if (ptx::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BM / 16; ++kk)
            ptx::mma2_ts(tbase + kDK, tbase + kDST + kk * 8, dQB + (uint64_t)(kk * 2048 >> 4), id_kd,
                         (i > 0 || kk > 0) ? 1u : 0u);
          ptx::mma2_commit(bar + B_QB_E);
        }
        __syncwarp();
      };
      ptx::mbar_wait(bar + B_KV, 0);
      ptx::mbar_wait(bar + B_QA_F, 0);
      ptx::tc_fence_after();
      st_mma();
      ptx::mbar_wait(bar + B_DA_F, 0);
      ptx::tc_fence_after();
      dpt_mma();
      for (int i = 0; i < nq; ++i) {
        const bool more = i + 1 < nq;
        // dV_i += P^T_i dO_i  (A = P^T in TMEM [0,64))
        ptx::mbar_wait(bar + B_P, i & 1); BTRACE6(0, i);
        ptx::mbar_wait(bar + B_DB_F, i & 1);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BM / 16; ++kk)
            ptx::mma2_ts(tbase + kDV, tbase + kS + kk * 8, dDOB + (uint64_t)(kk * 2048 >> 4), id_kd,
                         (i > 0 || kk > 0) ? 1u : 0u);
          ptx::mma2_commit(bar + B_DB_E);
        }
        __syncwarp();
        // S^T_{i+1}: the S region also holds dQ_{i-1} until it has been drained
        if (more) {
          if (i > 0) { ptx::mbar_wait(bar + B_DQE, (i - 1) & 1); BTRACE6(2, i); }
          ptx::mbar_wait(bar + B_QA_F, (i + 1) & 1); BTRACE6(11, i);
          ptx::tc_fence_after();
          st_mma();
        }
        // dK_i += dS^T_i Q_i, then dP^T_{i+1} over the dS^T columns dK_i just consumed
        ptx::mbar_wait(bar + B_DS, i & 1);
        ptx::mbar_wait(bar + B_QB_F, i & 1);
        BTRACE6(1, i);
        ptx::tc_fence_after();
        dk_mma(i);
        if (more) {
          ptx::mbar_wait(bar + B_DA_F, (i + 1) & 1); BTRACE6(10, i);
          ptx::tc_fence_after();
          dpt_mma();
        }
        // dQ_i = dS_i K over the pair's 256 keys into S columns [64,128): both dS halves
        // crossed over, and S^T_{i+1} already loaded by the P/dS warpgroups
        ptx::mbar_wait(bar + B_X, i & 1);     // peer's dS half landed here
        ptx::mbar_wait(bar + B_XR, i & 1);    // ... and ours landed in the peer (relayed)
        if (more) ptx::mbar_wait(bar + B_SREAD, (i + 1) & 1);
        BTRACE6(12, i);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < (2 * BN) / 16; ++kk)
            ptx::mma2_ss(tbase + kDQ, dDSQ + (uint64_t)(kk * 2048 >> 4),
                         dKQ + (uint64_t)(kk * 2048 >> 4), id_dq, kk > 0);
          ptx::mma2_commit(bar + B_DQF);
          ptx::mma2_commit(bar + B_DSQE);
        }
        __syncwarp();
      }
      if (ptx::elect_one()) ptx::mma2_commit(bar + B_DKV);
      __syncwarp();
    } else if (warp == 14 && lane == 0 && !leader && nq > 0) {
      // relay: tell the leader that the leader's dS half has landed in this CTA
      const uint32_t xr = ptx::leader_addr(bar + B_XR);
      for (int i = 0; i < nq; ++i) {
        ptx::mbar_wait(bar + B_X, i & 1);
        ptx::mbar_arrive_remote(xr);
      }
    }
  } else if (warp < 8) {
    // ------------------------------------------------------------ P / dS, query half hq
    ptx::regs_inc<144>();
    const int hq = warp >> 2;                  // query columns [64 hq, 64 hq + 64)
    const int t = threadIdx.x & 127;           // own key row = TMEM lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int64_t krow = k0 + t;
    const bool kvalid = krow < k_end && krow < hp.n_k;
    const int64_t kpos = (hp.causal || hp.grid_skip) ? pos_of(hp.k_map, kvalid ? krow : k0) : 0;
    const int64_t qfirst = hp.causal ? count_le(hp.q_map, hp.n_q, kpos - 1) : 0;
    const float c2 = p.scale_log2;
    const uint32_t p_bar = ptx::leader_addr(bar + B_P), ds_bar = ptx::leader_addr(bar + B_DS);
    const uint32_t sread_bar = ptx::leader_addr(bar + B_SREAD);
    // query half hq feeds the dQ of CTA hq: written locally when hq == crank, else
    // staged in XS and shipped to the peer's DSQ rows of this CTA's keys
    const bool local = hq == (int)crank;
    const uint32_t dsq_row = (uint32_t)(crank * BN + t);
    uint8_t* dst_row = local ? sm + L::DSQ + crank * 16384 + t * 128 : sm + L::XS + t * 128;
    const uint32_t xs_peer = ptx::peer_addr(sm + L::DSQ + crank * 16384, crank ^ 1u);
    const uint32_t xbar_peer = ptx::peer_addr(bar + B_X, crank ^ 1u);
    for (int i = 0; i < nq; ++i) {
      const int s = i % kStatSlots;
      const int64_t q0 = qtile(i) + 64 * hq;
      int64_t lo64 = qfirst - q0, hi64 = q_end - q0;
      const int lo = lo64 < 0 ? 0 : (lo64 > 64 ? 64 : (int)lo64);
      const int hi = !kvalid ? 0 : (hi64 > 64 ? 64 : (hi64 < 0 ? 0 : (int)hi64));
      uint64_t gq = 0;   // block-sparse grid: hidden query columns of this half
      if (hp.grid_skip) {
        const int nv = hi64 > 64 ? 64 : (hi64 < 0 ? 0 : (int)hi64);
        if (nv > 0) gq = grid_query_bits(hp, q0, nv, kpos);
      }
      const bool warp_full = __all_sync(0xffffffffu, lo == 0 && hi == 64 && gq == 0);
      ptx::mbar_wait(bar + B_ST_F + s, (i / kStatSlots) & 1);
      ptx::mbar_wait(bar + B_S, i & 1); if (hq == 0) BTRACE6(3, i);
      ptx::tc_fence_after();
      const float4* lse4 = reinterpret_cast<const float4*>(sStat + s * 256) + 16 * hq;
      const float4* dst4 = lse4 + BM / 4;
      float pr[64];
      {
        uint32_t r[64];
        ptx::tmem_ld32(tbase + lane_off + kS + 64 * hq, *reinterpret_cast<uint32_t(*)[32]>(r));
        ptx::tmem_ld32(tbase + lane_off + kS + 64 * hq + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
        ptx::tmem_wait_ld();
        ptx::reg_fence(r);
        // S^T_i is in registers in both warpgroups: P^T may now pack into [0,64) and
        // dQ_{i-1} (MMA issuer) may take [64,128)
        ptx::tc_fence_before();
        ptx::named_bar_sync(4, 2 * BN);
        ptx::mbar_arrive_to(sread_bar, leader, bar + B_SREAD);
#pragma unroll
        for (int c4 = 0; c4 < 16; ++c4) {
          const float4 Lv = lse4[c4];
          // x = S * scale*log2e - lse*log2e on packed fp32x2 (FFMA2)
          const float2 xa = ptx::ffma2(make_float2(__uint_as_float(r[4 * c4 + 0]), __uint_as_float(r[4 * c4 + 1])),
                                       make_float2(c2, c2), make_float2(-Lv.x, -Lv.y));
          const float2 xb = ptx::ffma2(make_float2(__uint_as_float(r[4 * c4 + 2]), __uint_as_float(r[4 * c4 + 3])),
                                       make_float2(c2, c2), make_float2(-Lv.z, -Lv.w));
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
        ptx::tmem_st32(tbase + lane_off + kS + 32 * hq, pk);   // P^T of half hq: [32 hq, +32)
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive_to(p_bar, leader, bar + B_P); if (hq == 0) BTRACE6(4, i);

      // dS = P (dP - D): read this half's dP^T, then (after both halves have read
      // theirs) write dS^T over [128,192) and dS to SMEM for the pair's dQ
      ptx::mbar_wait(bar + B_DP, i & 1); if (hq == 0) BTRACE6(5, i);
      ptx::tc_fence_after();
      uint32_t r[64];
      ptx::tmem_ld32(tbase + lane_off + kDP + 64 * hq, *reinterpret_cast<uint32_t(*)[32]>(r));
      ptx::tmem_ld32(tbase + lane_off + kDP + 64 * hq + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
      ptx::tmem_wait_ld();
      ptx::reg_fence(r);
      if (hq == 0) BTRACE6(13, i);
      ptx::tc_fence_before();
      ptx::named_bar_sync(2, 2 * BN);            // every dP^T column read before dS^T lands
      if (hq == 0) BTRACE6(14, i);
      uint32_t pk[32];
#pragma unroll
      for (int j4 = 0; j4 < 16; ++j4) {
        const float4 Dv = dst4[j4];
        const int c = 4 * j4;
        const float2 da = ptx::fmul2(make_float2(pr[c], pr[c + 1]),
                                     ptx::fadd2(make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])),
                                                make_float2(-Dv.x, -Dv.y)));
        const float2 db = ptx::fmul2(make_float2(pr[c + 2], pr[c + 3]),
                                     ptx::fadd2(make_float2(__uint_as_float(r[c + 2]), __uint_as_float(r[c + 3])),
                                                make_float2(-Dv.z, -Dv.w)));
        pk[2 * j4] = ptx::pack_bf16(da.x, da.y);
        pk[2 * j4 + 1] = ptx::pack_bf16(db.x, db.y);
      }
      ptx::tmem_st32(tbase + lane_off + kDST + 32 * hq, pk);
      ptx::mbar_wait(bar + B_DSQE, (i & 1) ^ 1);  // dQ_{i-1} retired: DSQ / XS free
      if (local && t == 0) ptx::mbar_expect_tx(bar + B_X, 16384);   // the peer's half of this tile
      // MN-major A rows of the dQ MMA: row = key, 64 queries (128 B, SW128)
#pragma unroll
      for (int ch = 0; ch < 8; ++ch)
        *reinterpret_cast<uint4*>(dst_row + ((ch ^ (dsq_row & 7)) << 4)) =
            make_uint4(pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2], pk[4 * ch + 3]);
      ptx::tmem_wait_st();
      if (hq == 0) BTRACE6(15, i);
      ptx::fence_proxy_async_smem();
      if (!local) {
        ptx::named_bar_sync(3, BN);
        if (t == 0)   // one TMA bulk copy ships this half: SMEM -> peer SMEM, tx on its B_X
          ptx::bulk_copy_to_peer(xs_peer, sm + L::XS, 16384, xbar_peer);
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive_to(ds_bar, leader, bar + B_DS); if (hq == 0) BTRACE6(6, i);
      ptx::mbar_arrive(bar + B_ST_E + s);
    }
    // -------------------------------------------------------- dK / dV epilogue
    if (nq > 0) {
      ptx::mbar_wait(bar + B_DKV, 0);
      ptx::tc_fence_after();
    }
    {
      float* dst = hq == 0 ? p.dv_acc : p.dk_acc;
      const float mul = hq == 0 ? 1.f : p.scale;
      const uint32_t col0 = hq == 0 ? kDV : kDK;
#pragma unroll 1
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t rr[32];
        if (nq > 0) {
          ptx::tmem_ld32(tbase + lane_off + col0 + cc * 32, rr);
          ptx::tmem_wait_ld();
          ptx::reg_fence(rr);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) rr[j] = 0u;
        }
        if (!kvalid) continue;
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float4* a = reinterpret_cast<float4*>(dst + tl_index(bh, krow, cc * 32 + j, D, NTk));
          float4 v = make_float4(__uint_as_float(rr[j]) * mul, __uint_as_float(rr[j + 1]) * mul,
                                 __uint_as_float(rr[j + 2]) * mul, __uint_as_float(rr[j + 3]) * mul);
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
    ptx::regs_dec<112>();
    // TMEM lane L holds query 64*crank + L%64, d columns 64*(L/64) + [0,64).  This
    // CTA's partial (64 queries x 128 d) is staged 8 column groups (32 d) at a time
    // and reduced with one TMA tensor reduction per step (tm_dq views the TL
    // workspace as [column group][128 rows][4 floats]; box = 8 groups x 64 rows).
    const int L = threadIdx.x & 127;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int dhalf = L >> 6, row = L & 63;
    const uint32_t dqe_bar = ptx::leader_addr(bar + B_DQE);
    float4* stg = reinterpret_cast<float4*>(sm + L::STAGE);
    for (int i = 0; i < nq; ++i) {
      const int64_t qrow0 = qtile(i) + crank * 64;
      const bool qvalid = qrow0 + row < q_end && qrow0 + row < hp.n_q;
      ptx::mbar_wait(bar + B_DQF, i & 1); BTRACE6(7, i);
      ptx::tc_fence_after();
      uint32_t r[64];
      ptx::tmem_ld32(tbase + lane_off + kDQ, *reinterpret_cast<uint32_t(*)[32]>(r));
      ptx::tmem_ld32(tbase + lane_off + kDQ + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
      ptx::tmem_wait_ld();
      ptx::reg_fence(r);
      ptx::tc_fence_before();
      ptx::mbar_arrive_to(dqe_bar, leader, bar + B_DQE); BTRACE6(8, i);
      const float sc = qvalid ? p.scale : 0.f;
#pragma unroll
      for (int step = 0; step < 4; ++step) {    // d columns [32 step, 32 step + 32)
        if (L == 0) ptx::bulk_wait_read<0>();   // staging consumed by the previous reductions
        ptx::named_bar_sync(1, 128);
        if (dhalf == (step >> 1)) {
          const int cbase = (step & 1) * 32;
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            const int c = cbase + 4 * g;
            stg[g * 64 + row] = make_float4(__uint_as_float(r[c]) * sc, __uint_as_float(r[c + 1]) * sc,
                                            __uint_as_float(r[c + 2]) * sc, __uint_as_float(r[c + 3]) * sc);
          }
        }
        ptx::fence_proxy_async_smem();
        ptx::named_bar_sync(1, 128);
        if (L == 0) {   // one 8 KB tensor reduction: 8 column groups x rows [64c, 64c+64)
          ptx::tma_reduce_add_3d(&p.tm_dq, stg, 0, (int)(crank * 64),
                                 (int)((bh * NTq + (qrow0 >> 7)) * (D / 4) + 8 * step));
          ptx::bulk_commit();
        }
      }
      BTRACE6(9, i);
    }
    if (L == 0) ptx::bulk_wait_all();
  }

  __syncwarp();
  ptx::tc_fence_before();
  ptx::cluster_sync();      // the peer may still write our DSQ / arrive on our barriers
  if (warp == 12) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_2sm(tbase, 512);
  }
}

}  // namespace bwd6
}  // namespace burst
