// LAO backward on sm_100a, K/V-stationary.
//
// Reference semantics: one call = ring.backward_step (ring.py:221-242) for every
// (batch, head) slice, i.e. local_backward (local_attn.py:255-289, tiled form
// _backward_tiled 313-353) over the hop's rectangle:
//     P = exp(S - lse); dV += P^T dO; dP = dO V^T; dS = P * (dP - D);
//     dQ += scale dS K;  dK += scale dS^T Q
// computed transposed per key tile (S^T = K Q^T), so the visiting block's dK/dV
// accumulate in TMEM across all query tiles and dQ (pinned on this rank) is
// reduced into an fp32 workspace with vector atomics.
//
// CTA = one key tile of 128 rows (K, V stationary in SMEM); loops over the
// hop's query tiles of 128 (Q_i, dO_i, lse_i, D_i double-buffered by TMA).
//   warps 0-3  P / dS warpgroup (thread = key row = TMEM lane); dK/dV epilogue
//   warps 4-7  dQ drain warpgroup (thread = query row of the dQ tile)
//   warp  8    TMA producer (+ TMEM allocator)
//   warp  9    tcgen05.mma issuer
// TMEM (512 cols for D=128): S^T [0,128) (P^T bf16 in [0,64)), dP^T [128,256)
// (then dQ_i once dS_i is built), dV [256,256+D), dK [256+D,256+2D).
#pragma once
#include <cuda.h>
#include "common.cuh"
#include "ptx.cuh"

namespace burst {
namespace bwd {

constexpr int BM = 128;  // query rows per iteration
constexpr int BN = 128;  // key rows per CTA
constexpr int kThreads = 384;   // 3 warpgroups (warps 10-11 idle) for setmaxnreg

template <int D>
struct Cfg {
  static constexpr int kBoxBytes = 128 * 64 * 2;
  static constexpr int kBoxes = D / 64;
  static constexpr int kTileBytes = kBoxBytes * kBoxes;    // K, V, Q_i, dO_i tiles
  static constexpr int kDsBytes = BN * BM * 2;              // dS^T tile (bf16)
  static constexpr int kStatBytes = 2 * BM * 4;             // lse2_i, D_i
  static constexpr int kPayload = 2 * kTileBytes + 2 * 2 * kTileBytes + kDsBytes + 2 * kStatBytes;
  static constexpr int kBarBytes = 128;
  static constexpr int kMaxSmem = 232448;
  static constexpr int kSmemBytes =
      (kPayload + kBarBytes + 1024 <= kMaxSmem) ? kPayload + kBarBytes + 1024 : kMaxSmem;
  static constexpr int kMaxPad = kSmemBytes - kPayload - kBarBytes;
};

struct Params {
  CUtensorMap tm_q, tm_k, tm_v, tm_do;
  const float* stats;    // [2][B*H][NTq*128]: lse*log2e, D
  float* dq_acc;         // TL over n_q
  float* dk_acc;         // TL over n_k
  float* dv_acc;
  burst_hop hop;
  float scale_log2, scale;
  int accumulate;
  long long* trace;   // BURST_TRACE builds only: per-iteration clock64 timeline
};

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          ptx::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(ptx::smem_u32(bar))
      : "memory");
}

#ifdef BURST_TRACE
#define BTRACE(ev, i)                                                                        \
  do {                                                                                       \
    if (p.trace && (blockIdx.x == 0 || blockIdx.x == 77) && blockIdx.y == 0 && blockIdx.z == 0 && \
        (i) < 64)                                                                            \
      p.trace[((blockIdx.x ? 16 : 0) + (ev)) * 64 + (i)] = clock64();                        \
  } while (0)
#else
#define BTRACE(ev, i)
#endif

template <int D>
__global__ void __launch_bounds__(kThreads, 1) lao_bwd_kernel(const __grid_constant__ Params p) {
  using C = Cfg<D>;
  // SW128 tiles need 1024-byte alignment; the declaration asks the compiler for it and
  // the runtime check below can then only fail on a toolchain that ignores it, in
  // which case the launch reports a CudaError (flag bit 2) instead of trapping.
  extern __shared__ __align__(1024) uint8_t smem_raw[];
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
  uint8_t* sdO = sQ + 2 * C::kTileBytes;       // [2] stages
  uint8_t* sdS = sdO + 2 * C::kTileBytes;
  float* sStat = reinterpret_cast<float*>(sdS + C::kDsBytes);   // [2][2][BM]
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
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 13);

  const burst_hop& hp = p.hop;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.z, h = blockIdx.y;
  const int64_t bh = (int64_t)b * hp.heads + h;
  const int64_t k0 = hp.k_begin + (int64_t)blockIdx.x * BN;   // first key row of this CTA
  const int64_t k_end = hp.k_begin + hp.k_len;
  const int64_t q_end = hp.q_begin + hp.q_len;
  const int64_t NTq = ceil_div(hp.n_q, 128);
  const int64_t NTk = ceil_div(hp.n_k, 128);

  // Query tiles touching this key tile: causal => suffix of the hop's queries.
  int64_t qs = hp.q_begin;
  if (hp.causal) {
    const int64_t first_q = count_le(hp.q_map, hp.n_q, pos_of(hp.k_map, k0) - 1);
    if (first_q > qs) qs = hp.q_begin + ((first_q - hp.q_begin) / BM) * BM;
  }
  const int nq = qs < q_end ? (int)ceil_div(q_end - qs, BM) : 0;
  // Query-tile visiting order is rotated per CTA: concurrently resident CTAs (consecutive
  // key tiles of one head) then reduce into different dQ tiles instead of all hitting
  // the same 64 KB of dQ_acc at once (L2 atomic hot spot).
  const int rot = nq > 0 ? (int)((blockIdx.x * 7u) % (unsigned)nq) : 0;
  auto qtile = [&](int i) -> int64_t { int j = i + rot; if (j >= nq) j -= nq; return qs + (int64_t)j * BM; };

  if (warp == 8) {
    if (lane == 0) {
      ptx::mbar_init(kv_full, 1);
      for (int s = 0; s < 2; ++s) {
        ptx::mbar_init(qdo_full + s, 1);
        ptx::mbar_init(qdo_empty + s, 1);
      }
      ptx::mbar_init(s_full, 1);
      ptx::mbar_init(p_full, BN);
      ptx::mbar_init(ds_full, BN);
      ptx::mbar_init(ds_empty, 1);
      ptx::mbar_init(dq_full, 1);
      ptx::mbar_init(dq_empty, BM);
      ptx::mbar_init(dkv_full, 1);
      ptx::mbar_init(dp_full, 1);
      ptx::fence_mbar_init();
      ptx::tma_prefetch_desc(&p.tm_q);
      ptx::tma_prefetch_desc(&p.tm_k);
      ptx::tma_prefetch_desc(&p.tm_v);
      ptx::tma_prefetch_desc(&p.tm_do);
    }
    __syncwarp();
    ptx::tmem_alloc(tmem_holder, 512);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = *tmem_holder;
  constexpr uint32_t kS = 0, kDP = 128, kDV = 256, kDK = 256 + D;
  if (warp >= 8) {
   ptx::regs_dec<88>();
   if (warp == 8) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && nq > 0) {
      ptx::mbar_expect_tx(kv_full, 2 * C::kTileBytes);
      for (int x = 0; x < C::kBoxes; ++x) {
        ptx::tma_load_4d(sK + x * C::kBoxBytes, &p.tm_k, kv_full, x * 64, h, (int)k0, b);
        ptx::tma_load_4d(sV + x * C::kBoxBytes, &p.tm_v, kv_full, x * 64, h, (int)k0, b);
      }
      for (int i = 0; i < nq; ++i) {
        const int s = i & 1;
        const int64_t q0 = qtile(i);
        ptx::mbar_wait(qdo_empty + s, ((i >> 1) & 1) ^ 1); BTRACE(10, i);
        ptx::mbar_expect_tx(qdo_full + s, 2 * C::kTileBytes + C::kStatBytes);
        for (int x = 0; x < C::kBoxes; ++x) {
          ptx::tma_load_4d(sQ + s * C::kTileBytes + x * C::kBoxBytes, &p.tm_q, qdo_full + s,
                           x * 64, h, (int)q0, b);
          ptx::tma_load_4d(sdO + s * C::kTileBytes + x * C::kBoxBytes, &p.tm_do, qdo_full + s,
                           x * 64, h, (int)q0, b);
        }
        const float* st = p.stats + bh * NTq * 128 + q0;
        bulk_load(sStat + s * 2 * BM, st, BM * 4, qdo_full + s);
        bulk_load(sStat + s * 2 * BM + BM, st + (int64_t)hp.batch * hp.heads * NTq * 128, BM * 4,
                  qdo_full + s);
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    // Order per query tile i (steady state):
    //   dV_i | S^T_{i+1} (overlaps dS_i) | dK_i, dQ_i -> dP region | dP^T_{i+1} (after dQ_i drained)
    if (lane == 0 && nq > 0) {
      constexpr uint32_t id_kk = ptx::make_idesc_bf16(BN, BM, 0, 0);   // S^T, dP^T
      constexpr uint32_t id_kmn = ptx::make_idesc_bf16(BN, D, 0, 1);   // dV, dK (B MN-major)
      constexpr uint32_t id_mnmn = ptx::make_idesc_bf16(BM, D, 1, 1);  // dQ (A, B MN-major)
      const uint32_t aK = ptx::smem_u32(sK), aV = ptx::smem_u32(sV);
      const uint32_t aQ = ptx::smem_u32(sQ), adO = ptx::smem_u32(sdO), adS = ptx::smem_u32(sdS);
      auto st_mma = [&](int stage) {   // S^T = K Q^T
        const uint32_t q = aQ + stage * C::kTileBytes;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * C::kBoxBytes + (kk & 3) * 32;
          ptx::mma_ss(tbase + kS, ptx::make_sdesc(aK + off, 0, 1024),
                      ptx::make_sdesc(q + off, 0, 1024), id_kk, kk > 0);
        }
      };
      auto dpt_mma = [&](int stage) {  // dP^T = V dO^T
        const uint32_t dO = adO + stage * C::kTileBytes;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * C::kBoxBytes + (kk & 3) * 32;
          ptx::mma_ss(tbase + kDP, ptx::make_sdesc(aV + off, 0, 1024),
                      ptx::make_sdesc(dO + off, 0, 1024), id_kk, kk > 0);
        }
      };
      ptx::mbar_wait(kv_full, 0);
      ptx::mbar_wait(qdo_full + 0, 0);
      ptx::tc_fence_after();
      st_mma(0);
      ptx::mma_commit(s_full);
      dpt_mma(0);
      ptx::mma_commit(dp_full);
      for (int i = 0; i < nq; ++i) {
        const int s = i & 1;
        const bool more = i + 1 < nq;
        const uint32_t q = aQ + s * C::kTileBytes, dO = adO + s * C::kTileBytes;
        // dV += P^T dO   (A = P^T from TMEM, B = dO MN-major, reduction over queries)
        ptx::mbar_wait(p_full, i & 1); BTRACE(0, i);
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BM / 16; ++kk)
          ptx::mma_ts(tbase + kDV, tbase + kS + kk * 8,
                      ptx::make_sdesc(dO + kk * 2048, C::kBoxBytes, 1024), id_kmn,
                      (i > 0 || kk > 0) ? 1u : 0u);
        if (more) {
          ptx::mbar_wait(qdo_full + (s ^ 1), ((i + 1) >> 1) & 1); BTRACE(11, i);
          ptx::tc_fence_after();
          st_mma(s ^ 1);
          ptx::mma_commit(s_full);
        }
        // dK += dS^T Q ; dQ_i = dS K  (into the dP^T columns, already consumed)
        ptx::mbar_wait(ds_full, i & 1); BTRACE(1, i);
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BM / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          ptx::mma_ss(tbase + kDK, ptx::make_sdesc(adS + off, 0, 1024),
                      ptx::make_sdesc(q + kk * 2048, C::kBoxBytes, 1024), id_kmn,
                      (i > 0 || kk > 0) ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk)
          ptx::mma_ss(tbase + kDP, ptx::make_sdesc(adS + kk * 2048, 16384, 1024),
                      ptx::make_sdesc(aK + kk * 2048, C::kBoxBytes, 1024), id_mnmn, kk > 0);
        ptx::mma_commit(dq_full);
        ptx::mma_commit(ds_empty);
        ptx::mma_commit(qdo_empty + s);
        if (more) {
          ptx::mbar_wait(dq_empty, i & 1); BTRACE(2, i);
          ptx::tc_fence_after();
          dpt_mma(s ^ 1);
          ptx::mma_commit(dp_full);
        }
      }
      ptx::mma_commit(dkv_full);
    }
   }
  } else if (warp < 4) {
    // ------------------------------------------------------------ P / dS warpgroup
    ptx::regs_inc<240>();
    const int t = threadIdx.x;                  // key row within the tile
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int64_t krow = k0 + t;
    const bool kvalid = krow < k_end && krow < hp.n_k;
    const int64_t kpos = (hp.causal || hp.grid_skip) ? pos_of(hp.k_map, kvalid ? krow : k0) : 0;
    const int64_t qfirst = hp.causal ? count_le(hp.q_map, hp.n_q, kpos - 1) : 0;
    const float c2 = p.scale_log2;
    for (int i = 0; i < nq; ++i) {
      const int s = i & 1;
      const int64_t q0 = qtile(i);
      // visible query columns of this key row: [lo, hi)
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
      ptx::mbar_wait(qdo_full + s, (i >> 1) & 1);
      ptx::mbar_wait(s_full, i & 1); BTRACE(3, i);
      ptx::tc_fence_after();
      const float4* lse4 = reinterpret_cast<const float4*>(sStat + s * 2 * BM);
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
          const float4 L = lse4[c4];
          pr[4 * c4 + 0] = ptx::ex2(fmaf(__uint_as_float(r[4 * c4 + 0]), c2, -L.x));
          pr[4 * c4 + 1] = ptx::ex2(fmaf(__uint_as_float(r[4 * c4 + 1]), c2, -L.y));
          pr[4 * c4 + 2] = ptx::ex2(fmaf(__uint_as_float(r[4 * c4 + 2]), c2, -L.z));
          pr[4 * c4 + 3] = ptx::ex2(fmaf(__uint_as_float(r[4 * c4 + 3]), c2, -L.w));
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
      ptx::mbar_arrive(p_full); BTRACE(4, i);

      ptx::mbar_wait(dp_full, i & 1); BTRACE(5, i);
      ptx::mbar_wait(ds_empty, (i & 1) ^ 1);
      ptx::tc_fence_after();
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t r[64];
        ptx::tmem_ld32(tbase + lane_off + kDP + half * 64, *reinterpret_cast<uint32_t(*)[32]>(r));
        ptx::tmem_ld32(tbase + lane_off + kDP + half * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
        ptx::tmem_wait_ld();
        ptx::reg_fence(r);
        uint32_t pk[32];
#pragma unroll
        for (int j4 = 0; j4 < 16; ++j4) {
          const float4 Dv = dst4[half * 16 + j4];
          const int c = half * 64 + 4 * j4;
          // masked entries (P = 0) give dS = 0 exactly: a query tile that starts off the
          // 128-row grid reads up to 127 lse/D values past the hop's last row (the next
          // head's statistics, or past the end of the buffer for the last head), and
          // 0 * (dP - garbage) must not turn into NaN
          auto ds = [](float pv, float dp, float dd) { return pv != 0.f ? pv * (dp - dd) : 0.f; };
          pk[2 * j4] = ptx::pack_bf16(ds(pr[c], __uint_as_float(r[4 * j4]), Dv.x),
                                      ds(pr[c + 1], __uint_as_float(r[4 * j4 + 1]), Dv.y));
          pk[2 * j4 + 1] = ptx::pack_bf16(ds(pr[c + 2], __uint_as_float(r[4 * j4 + 2]), Dv.z),
                                          ds(pr[c + 3], __uint_as_float(r[4 * j4 + 3]), Dv.w));
        }
        // SW128 K-major: row t, 16-byte query chunk ch (8 bf16) of 128 B swizzle row
        uint8_t* rowp = sdS + half * 16384 + t * 128;
#pragma unroll
        for (int ch = 0; ch < 8; ++ch)
          *reinterpret_cast<uint4*>(rowp + ((ch ^ (t & 7)) << 4)) =
              make_uint4(pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2], pk[4 * ch + 3]);
      }
      ptx::fence_proxy_async_smem();
      ptx::tc_fence_before();
      ptx::mbar_arrive(ds_full); BTRACE(6, i);
    }
    // -------------------------------------------------------- dK / dV epilogue
    if (nq > 0) {
      ptx::mbar_wait(dkv_full, 0);
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
    const int t = threadIdx.x & 127;           // query row within the tile
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    for (int i = 0; i < nq; ++i) {
      const int64_t qrow = qtile(i) + t;
      const bool qvalid = qrow < q_end && qrow < hp.n_q;
      ptx::mbar_wait(dq_full, i & 1); BTRACE(7, i);
      ptx::tc_fence_after();
      uint32_t r[D];
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc)
        ptx::tmem_ld32(tbase + lane_off + kDP + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(r + cc * 32));
      ptx::tmem_wait_ld();
      ptx::reg_fence(r);
      ptx::tc_fence_before();
      ptx::mbar_arrive(dq_empty); BTRACE(8, i);
      if (qvalid) {
        float* base = p.dq_acc + tl_index(bh, qrow, 0, D, NTq);
#pragma unroll
        for (int j = 0; j < D; j += 4)   // next 4-column group: 128 rows x 4 floats further
          ptx::red_add_v4(base + (size_t)(j >> 2) * 512, __uint_as_float(r[j]) * p.scale,
                          __uint_as_float(r[j + 1]) * p.scale, __uint_as_float(r[j + 2]) * p.scale,
                          __uint_as_float(r[j + 3]) * p.scale);
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

}  // namespace bwd
}  // namespace burst
