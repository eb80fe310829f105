// LAO forward on sm_100a with 64-key tiles and a double-buffered score tile per
// query tile, head_dim 128.
//
// Why (profiles/r01_trace_fwd*.txt): in lao_fwd (128-key tiles) the next score tile
// S_t(j+1) overwrites the TMEM columns holding P_t(j), so QK_t(j+1) can only be
// issued after PV_t(j): every step pays softmax_t(j) -> PV -> QK -> softmax_t(j+1),
// ~1300 cycles of MMA latency on the softmax warps' critical path (~3400 cycles per
// 128 keys, 63% tensor-pipe utilisation).  With 64-key tiles TMEM holds TWO score
// buffers per query tile (4 x 64 + 2 x 128 O columns = 512), so QK_t(j+1) runs while
// softmax_t(j) works and the softmax warpgroups go from one step to the next
// without waiting on the tensor pipe.
//
// Reference semantics as lao_fwd: one call = ring.forward_step (ring.py:158-181):
// local_forward_tiled (local_attn.py:207-248) + PartialAttn.merge (101-120), and on
// the last hop PartialAttn.finalize (127-135).  Dense hops only (grid-masked hops use
// lao_fwd).
//
// CTA = 2 query tiles x 128 rows sharing every K/V tile (64 keys, 8-stage TMA ring).
//   warps 0-3  softmax/epilogue for query tile 0 (thread = row = TMEM lane)
//   warps 4-7  softmax/epilogue for query tile 1
//   warp  8    TMA producer (+ TMEM allocator);  warp 9 MMA issuer (whole warp, elected lane)
// TMEM: S[t][b] at t*128 + b*64 (64 fp32 columns; P[t][b] bf16 in its first 32),
//       O[t] at 256 + t*128.
// MMA order per KV step j: QK_0(j+1), QK_1(j+1) | PV_0(j) | PV_1(j).
#pragma once
#include <cuda.h>
#include "common.cuh"
#include "ptx.cuh"

namespace burst {
namespace fwd2 {

constexpr int D = 128;
constexpr int BM = 128;        // query rows per tile
constexpr int BN = 64;         // keys per tile
constexpr int kThreads = 384;
constexpr int kStages = 8;     // K / V half tiles in flight
constexpr float kRescaleThreshold = 8.0f;
constexpr int kQBox = 128 * 64 * 2;     // Q: 128 rows x 64 d
constexpr int kQTile = 2 * kQBox;       // 32 KB
constexpr int kKVBox = 64 * 64 * 2;     // K/V: 64 rows x 64 d
constexpr int kKVTile = 2 * kKVBox;     // 16 KB
constexpr int kSmemBytes = 1024 + 2 * kQTile + kStages * kKVTile + 256;

struct Params {
  CUtensorMap tm_q, tm_k, tm_v;   // tm_k / tm_v boxes of 64 rows
  float* o_acc;
  float* m_run;
  float* l_run;
  void* o_out;
  float* lse_out;
  int* flags;
  burst_hop hop;
  float scale_log2;
  int first_hop, finalize;
};

__global__ void __launch_bounds__(kThreads, 1) lao_fwd2_kernel(const __grid_constant__ Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem;
  {
    const uint32_t s = ptx::smem_u32(smem_raw);
    smem = smem_raw + ((1024u - (s & 1023u)) & 1023u);
  }
  uint8_t* sQ = smem;                       // 2 tiles
  uint8_t* sKV = smem + 2 * kQTile;         // kStages slots (K_j, V_j alternate)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + kStages * kKVTile);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + kStages;
  uint64_t* s_full = kv_empty + kStages;    // [t][b]
  uint64_t* p_full = s_full + 4;            // [t][b]
  uint64_t* o_done = p_full + 4;            // [t]: PV_t(j) retired (lazy-rescale guard)
  uint64_t* o_full = o_done + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(o_full + 1);

  const burst_hop& hp = p.hop;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.z, h = blockIdx.y;
  const int64_t q_end = hp.q_begin + hp.q_len;
  const int64_t xb = hp.causal ? (int64_t)(gridDim.x - 1 - blockIdx.x) : (int64_t)blockIdx.x;
  const int64_t row0 = hp.q_begin + xb * (2 * BM);

  int64_t kspan = hp.k_len;
  if (hp.causal) {
    int64_t last = (row0 + 2 * BM < q_end ? row0 + 2 * BM : q_end) - 1;
    int64_t cnt = count_le(hp.k_map, hp.n_k, pos_of(hp.q_map, last)) - hp.k_begin;
    kspan = cnt < kspan ? cnt : kspan;
    if (kspan < 0) kspan = 0;
  }
  const int nkv = (int)ceil_div(kspan, BN);

  if (warp == 8) {
    if (lane == 0) {
      ptx::mbar_init(q_full, 1);
      for (int s = 0; s < kStages; ++s) {
        ptx::mbar_init(kv_full + s, 1);
        ptx::mbar_init(kv_empty + s, 1);
      }
      for (int i = 0; i < 4; ++i) {
        ptx::mbar_init(s_full + i, 1);
        ptx::mbar_init(p_full + i, BM);
      }
      ptx::mbar_init(o_done + 0, 1);
      ptx::mbar_init(o_done + 1, 1);
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
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = *tmem_holder;
  if (warp >= 8) {
   ptx::regs_dec<88>();
   if (warp == 8) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && nkv > 0) {
      ptx::mbar_expect_tx(q_full, 2 * kQTile);
      for (int t = 0; t < 2; ++t)
        for (int x = 0; x < 2; ++x)
          ptx::tma_load_4d(sQ + t * kQTile + x * kQBox, &p.tm_q, q_full, x * 64, h,
                           (int)(row0 + t * BM), b);
      int it = 0;
      for (int j = 0; j < nkv; ++j) {
        const int krow = (int)(hp.k_begin + (int64_t)j * BN);
        for (int kv = 0; kv < 2; ++kv, ++it) {
          const int s = it % kStages;
          const uint32_t use = it / kStages;
          ptx::mbar_wait(kv_empty + s, (use & 1) ^ 1);
          ptx::mbar_expect_tx(kv_full + s, kKVTile);
          const CUtensorMap* tm = kv == 0 ? &p.tm_k : &p.tm_v;
          for (int x = 0; x < 2; ++x)
            ptx::tma_load_4d(sKV + s * kKVTile + x * kKVBox, tm, kv_full + s, x * 64, h, krow, b);
        }
      }
    }
   } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    if (nkv > 0) {
      constexpr uint32_t idesc_qk = ptx::make_idesc_bf16(BM, BN, 0, 0);
      constexpr uint32_t idesc_pv = ptx::make_idesc_bf16(BM, D, 0, 1);
      const uint64_t dQk = ptx::make_sdesc(ptx::smem_u32(sQ), 0, 1024);
      const uint64_t dKVk = ptx::make_sdesc(ptx::smem_u32(sKV), 0, 1024);       // K (K-major)
      const uint64_t dKVm = ptx::make_sdesc(ptx::smem_u32(sKV), kKVBox, 1024);  // V (MN-major)
      constexpr uint64_t kQT = (uint64_t)(kQTile >> 4), kKVT = (uint64_t)(kKVTile >> 4);
      auto qk = [&](int t, int slot, int buf) {   // S[t][buf] = Q_t K^T
        if (ptx::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t oq = (uint64_t)(((kk >> 2) * kQBox + (kk & 3) * 32) >> 4);
            const uint64_t ok = (uint64_t)(((kk >> 2) * kKVBox + (kk & 3) * 32) >> 4);
            ptx::mma_ss(tbase + t * 128 + buf * 64, dQk + t * kQT + oq, dKVk + slot * kKVT + ok,
                        idesc_qk, kk > 0);
          }
          ptx::mma_commit(s_full + 2 * t + buf);
        }
        __syncwarp();
      };
      auto pv = [&](int t, int slot, int buf, bool acc) {   // O[t] += P[t][buf] V
        if (ptx::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk)
            ptx::mma_ts(tbase + 256 + t * 128, tbase + t * 128 + buf * 64 + kk * 8,
                        dKVm + slot * kKVT + (uint64_t)(kk * 2048 >> 4), idesc_pv,
                        (acc || kk > 0) ? 1u : 0u);
          ptx::mma_commit(o_done + t);
        }
        __syncwarp();
      };
      auto commit = [&](uint64_t* bb) {
        if (ptx::elect_one()) ptx::mma_commit(bb);
        __syncwarp();
      };
      ptx::mbar_wait(q_full, 0);
      ptx::mbar_wait(kv_full + 0, 0);
      ptx::tc_fence_after();
      qk(0, 0, 0);
      qk(1, 0, 0);
      commit(kv_empty + 0);
      for (int j = 0; j < nkv; ++j) {
        const int b0 = j & 1;
        const int itv = 2 * j + 1, sv = itv % kStages;
        if (j + 1 < nkv) {      // next scores first: they land in the other buffer
          const int itk = 2 * j + 2, sk = itk % kStages;
          ptx::mbar_wait(kv_full + sk, (itk / kStages) & 1);
          ptx::tc_fence_after();
          qk(0, sk, b0 ^ 1);
          qk(1, sk, b0 ^ 1);
          commit(kv_empty + sk);
        }
        ptx::mbar_wait(kv_full + sv, (itv / kStages) & 1);
        ptx::mbar_wait(p_full + 0 + b0, (j >> 1) & 1);
        ptx::tc_fence_after();
        pv(0, sv, b0, j > 0);
        ptx::mbar_wait(p_full + 2 + b0, (j >> 1) & 1);
        ptx::tc_fence_after();
        pv(1, sv, b0, j > 0);
        commit(kv_empty + sv);
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
    const uint32_t tO = tbase + lane_off + 256 + g * 128;
    const int64_t row = row0 + g * BM + t;
    const bool valid = row < q_end && row < hp.n_q;
    int64_t lim = hp.k_len;
    if (hp.causal) {
      int64_t cnt = count_le(hp.k_map, hp.n_k, pos_of(hp.q_map, valid ? row : q_end - 1)) -
                    hp.k_begin;
      lim = cnt < lim ? cnt : lim;
    }
    const float c2 = p.scale_log2;
    float m_run = -INFINITY, l_run = 0.f;

    for (int j = 0; j < nkv; ++j) {
      const int b0 = j & 1;
      const uint32_t tS = tbase + lane_off + g * 128 + b0 * 64;
      ptx::mbar_wait(s_full + 2 * g + b0, (j >> 1) & 1);
      ptx::tc_fence_after();
      float s[BN];
      {
        uint32_t r[BN];
        ptx::tmem_ld32(tS, *reinterpret_cast<uint32_t(*)[32]>(r));
        ptx::tmem_ld32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
        ptx::tmem_wait_ld();
        ptx::reg_fence(r);
#pragma unroll
        for (int i = 0; i < BN; ++i) s[i] = __uint_as_float(r[i]);
      }
      const int64_t nvalid = lim - (int64_t)j * BN;
      if (__any_sync(0xffffffffu, nvalid < BN)) {
#pragma unroll
        for (int i = 0; i < BN; ++i)
          if (i >= nvalid) s[i] = -INFINITY;
      }
      float mx8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mx8[u] = s[u];
#pragma unroll
      for (int i = 8; i < BN; ++i) mx8[i & 7] = fmaxf(mx8[i & 7], s[i]);
      const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                             fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      const float m_tile = mx * c2;
      const bool grow = m_tile > m_run + kRescaleThreshold || (m_run == -INFINITY && m_tile > -INFINITY);
      if (__any_sync(0xffffffffu, grow && j > 0)) {
        // O[g] may still be accumulating PV_g(j-1): wait for it before rescaling
        ptx::mbar_wait(o_done + g, (j - 1) & 1);
        ptx::tc_fence_after();
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
        ptx::tmem_wait_st();
        l_run *= alpha;
        m_run = m_new;
      } else if (grow) {
        m_run = fmaxf(m_tile, m_run);
      }
      const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
      float2 ls4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                       make_float2(0.f, 0.f)};
      const float2 c2v = make_float2(c2, c2), negm = make_float2(-m_use, -m_use);
      uint32_t pk[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float2 x = ptx::ffma2(make_float2(s[2 * i], s[2 * i + 1]), c2v, negm);
        const float p0 = ptx::ex2(x.x), p1 = ptx::ex2(x.y);
        ls4[i & 3] = ptx::fadd2(ls4[i & 3], make_float2(p0, p1));
        pk[i] = ptx::pack_bf16(p0, p1);
      }
      ptx::tmem_st32(tS, pk);
      const float2 lsa = ptx::fadd2(ptx::fadd2(ls4[0], ls4[1]), ptx::fadd2(ls4[2], ls4[3]));
      l_run += lsa.x + lsa.y;
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive(p_full + 2 * g + b0);
    }

    // ------------------------------------------------------------ epilogue (as lao_fwd)
    if (nkv > 0) {
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
    if (valid && p.finalize && !(l_new > 0.f)) atomicOr(p.flags, 1);
#pragma unroll
    for (int cc = 0; cc < D / 32; ++cc) {
      uint32_t r[32];
      if (nkv > 0) {
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
        p.lse_out[bh * hp.n_q + row] = (l_new > 0.f) ? (m_new + __log2f(l_new)) * kLn2 : -INFINITY;
      } else {
        p.m_run[bh * hp.n_q + row] = m_new;
        p.l_run[bh * hp.n_q + row] = l_new;
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

}  // namespace fwd2
}  // namespace burst
