// fp32 LAO forward/backward on CUDA cores (the reference's `precision="single"`
// path, BASELINE config C1).  tcgen05 has no fp32 kind (tf32 would miss the
// 1e-5 relative bar), so this is the f32 specialisation of the same hop
// contract as the sm_100a bf16 kernels: same running state, same TL
// workspaces, same masks.  Head dim <= 64.
//
// Reference: local_forward_tiled (local_attn.py:207-248) + merge (101-120) +
// finalize (127-135); local_backward (local_attn.py:255-289).
#pragma once
#include "common.cuh"

namespace burst {
namespace simt {

constexpr int kRows = 128;   // rows (threads) per CTA
constexpr int kTile = 32;    // keys / queries staged per SMEM tile

struct FwdParams {
  const float* q;
  const float* k;
  const float* v;
  float* o_acc;
  float* m_run;
  float* l_run;
  float* o_out;
  float* lse_out;
  int* flags;
  burst_hop hop;
  float scale_log2;
  int first_hop, finalize;
};

// Forward: thread = query row; K/V tiles of 32 keys staged in SMEM.
template <int D>
__global__ void __launch_bounds__(kRows) simt_fwd_kernel(const FwdParams p) {
  __shared__ float sk[kTile][D + 1];
  __shared__ float sv[kTile][D + 1];
  const burst_hop& hp = p.hop;
  const int b = blockIdx.z, h = blockIdx.y, t = threadIdx.x;
  const int64_t q_end = hp.q_begin + hp.q_len;
  const int64_t row0 = hp.q_begin + (int64_t)blockIdx.x * kRows;
  const int64_t row = row0 + t;
  const bool valid = row < q_end;
  const int64_t bh = (int64_t)b * hp.heads + h;
  const int64_t qpos = pos_of(hp.q_map, valid ? row : (q_end > 0 ? q_end - 1 : 0));

  int64_t kspan = hp.k_len, lim = hp.k_len;
  if (hp.causal) {
    const int64_t last = (row0 + kRows < q_end ? row0 + kRows : q_end) - 1;
    int64_t c = count_le(hp.k_map, hp.n_k, pos_of(hp.q_map, last)) - hp.k_begin;
    kspan = c < kspan ? c : kspan;
    c = count_le(hp.k_map, hp.n_k, pos_of(hp.q_map, valid ? row : last)) - hp.k_begin;
    lim = c < lim ? c : lim;
  }
  float q[D], o[D];
#pragma unroll
  for (int c = 0; c < D; ++c) {
    q[c] = valid ? p.q[(((int64_t)b * hp.n_q + row) * hp.heads + h) * D + c] : 0.f;
    o[c] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  for (int64_t k0 = 0; k0 < kspan; k0 += kTile) {
    __syncthreads();
    for (int e = t; e < kTile * D; e += kRows) {
      const int r = e / D, c = e % D;
      const int64_t kr = hp.k_begin + k0 + r;
      const bool ok = kr < hp.n_k;
      const int64_t gi = (((int64_t)b * hp.n_k + kr) * hp.heads + h) * D + c;
      sk[r][c] = ok ? p.k[gi] : 0.f;
      sv[r][c] = ok ? p.v[gi] : 0.f;
    }
    __syncthreads();
    float s[kTile];
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < kTile; ++j) {
      float acc = 0.f;
#pragma unroll
      for (int c = 0; c < D; ++c) acc = fmaf(q[c], sk[j][c], acc);
      const bool hidden = k0 + j >= lim ||
          (hp.grid_skip && grid_skipped(hp, qpos, pos_of(hp.k_map, hp.k_begin + k0 + j)));
      s[j] = hidden ? -INFINITY : acc * p.scale_log2;
      mx = fmaxf(mx, s[j]);
    }
    const float m_new = fmaxf(m, mx);
    if (m_new > m) {
      const float alpha = (m == -INFINITY) ? 0.f : exp2f(m - m_new);
      l *= alpha;
#pragma unroll
      for (int c = 0; c < D; ++c) o[c] *= alpha;
      m = m_new;
    }
    const float m_use = (m == -INFINITY) ? 0.f : m;
#pragma unroll
    for (int j = 0; j < kTile; ++j) {
      const float pj = exp2f(s[j] - m_use);
      l += pj;
#pragma unroll
      for (int c = 0; c < D; ++c) o[c] = fmaf(pj, sv[j][c], o[c]);
    }
  }
  if (!valid) return;
  const int64_t NT = ceil_div(hp.n_q, 128);
  float m_old = -INFINITY, l_old = 0.f;
  if (!p.first_hop) {
    m_old = p.m_run[bh * hp.n_q + row];
    l_old = p.l_run[bh * hp.n_q + row];
  }
  const float mn = fmaxf(m_old, m);
  const float a_old = (m_old == -INFINITY) ? 0.f : exp2f(m_old - mn);
  const float a_hop = (m == -INFINITY) ? 0.f : exp2f(m - mn);
  const float ln = a_old * l_old + a_hop * l;
  if (p.finalize && ln == 0.f) atomicOr(p.flags, 1);   // MaskError
  float nf = 0.f;                                      // NaN iff an output is non-finite
  const float inv = ln > 0.f ? 1.f / ln : 0.f;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const size_t ti = tl_index(bh, row, c, D, NT);
    const float prev = p.first_hop ? 0.f : p.o_acc[ti];
    const float val = a_old * prev + a_hop * o[c];
    if (p.finalize) {
      p.o_out[(((int64_t)b * hp.n_q + row) * hp.heads + h) * D + c] = val * inv;
      nf = fmaf(val * inv, 0.f, nf);
    }
    else
      p.o_acc[ti] = val;
  }
  if (p.finalize) {
    const float lse = ln > 0.f ? (mn + log2f(ln)) * kLn2 : -INFINITY;
    p.lse_out[bh * hp.n_q + row] = lse;
    if (ln != 0.f && !(fabsf(nf + lse) <= 3.0e38f)) atomicOr(p.flags, 2);   // NonFiniteError
  } else {
    p.m_run[bh * hp.n_q + row] = mn;
    p.l_run[bh * hp.n_q + row] = ln;
  }
}

struct BwdParams {
  const float* q;
  const float* k;
  const float* v;
  const float* dout;
  const float* stats;   // [2][B*H][NTq*128]: lse*log2e, D
  float* dq_acc;
  float* dk_acc;
  float* dv_acc;
  burst_hop hop;
  float scale_log2, scale;
  int accumulate;
};

// dQ: thread = query row, loop over visible keys (recomputes P; no atomics).
template <int D>
__global__ void __launch_bounds__(kRows) simt_bwd_dq_kernel(const BwdParams p) {
  __shared__ float sk[kTile][D + 1];
  __shared__ float sv[kTile][D + 1];
  const burst_hop& hp = p.hop;
  const int b = blockIdx.z, h = blockIdx.y, t = threadIdx.x;
  const int64_t q_end = hp.q_begin + hp.q_len;
  const int64_t row0 = hp.q_begin + (int64_t)blockIdx.x * kRows;
  const int64_t row = row0 + t;
  const bool valid = row < q_end;
  const int64_t bh = (int64_t)b * hp.heads + h;
  const int64_t NTq = ceil_div(hp.n_q, 128);
  const int64_t qpos = pos_of(hp.q_map, valid ? row : (q_end > 0 ? q_end - 1 : 0));
  int64_t kspan = hp.k_len, lim = hp.k_len;
  if (hp.causal) {
    const int64_t last = (row0 + kRows < q_end ? row0 + kRows : q_end) - 1;
    int64_t c = count_le(hp.k_map, hp.n_k, pos_of(hp.q_map, last)) - hp.k_begin;
    kspan = c < kspan ? c : kspan;
    c = count_le(hp.k_map, hp.n_k, pos_of(hp.q_map, valid ? row : last)) - hp.k_begin;
    lim = c < lim ? c : lim;
  }
  float q[D], dO[D], dq[D];
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const int64_t gi = (((int64_t)b * hp.n_q + row) * hp.heads + h) * D + c;
    q[c] = valid ? p.q[gi] : 0.f;
    dO[c] = valid ? p.dout[gi] : 0.f;
    dq[c] = 0.f;
  }
  const float lse2 = valid ? p.stats[bh * NTq * 128 + row] : INFINITY;
  const float dst = valid ? p.stats[((int64_t)hp.batch * hp.heads + bh) * NTq * 128 + row] : 0.f;
  for (int64_t k0 = 0; k0 < kspan; k0 += kTile) {
    __syncthreads();
    for (int e = t; e < kTile * D; e += kRows) {
      const int r = e / D, c = e % D;
      const int64_t kr = hp.k_begin + k0 + r;
      const bool ok = kr < hp.n_k;
      const int64_t gi = (((int64_t)b * hp.n_k + kr) * hp.heads + h) * D + c;
      sk[r][c] = ok ? p.k[gi] : 0.f;
      sv[r][c] = ok ? p.v[gi] : 0.f;
    }
    __syncthreads();
#pragma unroll 4
    for (int j = 0; j < kTile; ++j) {
      if (k0 + j >= lim) continue;
      if (hp.grid_skip && grid_skipped(hp, qpos, pos_of(hp.k_map, hp.k_begin + k0 + j))) continue;
      float s = 0.f, dp = 0.f;
#pragma unroll
      for (int c = 0; c < D; ++c) {
        s = fmaf(q[c], sk[j][c], s);
        dp = fmaf(dO[c], sv[j][c], dp);
      }
      const float pj = exp2f(s * p.scale_log2 - lse2);
      const float ds = pj * (dp - dst);
#pragma unroll
      for (int c = 0; c < D; ++c) dq[c] = fmaf(ds, sk[j][c], dq[c]);
    }
  }
  if (!valid) return;
#pragma unroll
  for (int c = 0; c < D; ++c) p.dq_acc[tl_index(bh, row, c, D, NTq)] += dq[c] * p.scale;
}

// dK/dV: thread = key row, loop over visible queries (Q, dO, lse, D staged in SMEM).
template <int D>
__global__ void __launch_bounds__(kRows) simt_bwd_dkv_kernel(const BwdParams p) {
  __shared__ float sq[kTile][D + 1];
  __shared__ float sdo[kTile][D + 1];
  __shared__ float sl[kTile], sd[kTile];
  extern __shared__ float acc_smem[];   // [2][kRows][D+1]: dK, dV accumulators
  const burst_hop& hp = p.hop;
  const int b = blockIdx.z, h = blockIdx.y, t = threadIdx.x;
  const int64_t k_end = hp.k_begin + hp.k_len;
  const int64_t q_end = hp.q_begin + hp.q_len;
  const int64_t k0 = hp.k_begin + (int64_t)blockIdx.x * kRows;
  const int64_t krow = k0 + t;
  const bool valid = krow < k_end;
  const int64_t bh = (int64_t)b * hp.heads + h;
  const int64_t NTq = ceil_div(hp.n_q, 128);
  const int64_t NTk = ceil_div(hp.n_k, 128);
  float* dk = acc_smem + t * (D + 1);
  float* dv = acc_smem + (kRows + t) * (D + 1);
  int64_t qs = hp.q_begin, qfirst = hp.q_begin;
  if (hp.causal) {
    const int64_t f = count_le(hp.q_map, hp.n_q, pos_of(hp.k_map, k0) - 1);
    qs = f > qs ? f : qs;
    const int64_t g = count_le(hp.q_map, hp.n_q, pos_of(hp.k_map, valid ? krow : k0) - 1);
    qfirst = g > qfirst ? g : qfirst;
  }
  const int64_t kposg = pos_of(hp.k_map, valid ? krow : k0);
  float kr[D], vr[D];
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const int64_t gi = (((int64_t)b * hp.n_k + krow) * hp.heads + h) * D + c;
    kr[c] = valid ? p.k[gi] : 0.f;
    vr[c] = valid ? p.v[gi] : 0.f;
    dk[c] = 0.f;
    dv[c] = 0.f;
  }
  for (int64_t q0 = qs; q0 < q_end; q0 += kTile) {
    __syncthreads();
    for (int e = t; e < kTile * D; e += kRows) {
      const int r = e / D, c = e % D;
      const int64_t qr = q0 + r;
      const bool ok = qr < q_end;
      const int64_t gi = (((int64_t)b * hp.n_q + qr) * hp.heads + h) * D + c;
      sq[r][c] = ok ? p.q[gi] : 0.f;
      sdo[r][c] = ok ? p.dout[gi] : 0.f;
    }
    if (t < kTile) {
      const int64_t qr = q0 + t;
      const bool ok = qr < q_end;
      sl[t] = ok ? p.stats[bh * NTq * 128 + qr] : INFINITY;
      sd[t] = ok ? p.stats[((int64_t)hp.batch * hp.heads + bh) * NTq * 128 + qr] : 0.f;
    }
    __syncthreads();
    if (!valid) continue;
    for (int j = 0; j < kTile; ++j) {
      if (q0 + j < qfirst || q0 + j >= q_end) continue;
      if (hp.grid_skip && grid_skipped(hp, pos_of(hp.q_map, q0 + j), kposg)) continue;
      float s = 0.f, dp = 0.f;
#pragma unroll
      for (int c = 0; c < D; ++c) {
        s = fmaf(sq[j][c], kr[c], s);
        dp = fmaf(sdo[j][c], vr[c], dp);
      }
      const float pj = exp2f(s * p.scale_log2 - sl[j]);
      const float ds = pj * (dp - sd[j]);
#pragma unroll
      for (int c = 0; c < D; ++c) {
        dv[c] = fmaf(pj, sdo[j][c], dv[c]);
        dk[c] = fmaf(ds, sq[j][c], dk[c]);
      }
    }
  }
  if (!valid) return;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const size_t ti = tl_index(bh, krow, c, D, NTk);
    const float a = dk[c] * p.scale, bv = dv[c];
    if (p.accumulate) {
      p.dk_acc[ti] += a;
      p.dv_acc[ti] += bv;
    } else {
      p.dk_acc[ti] = a;
      p.dv_acc[ti] = bv;
    }
  }
}

}  // namespace simt
}  // namespace burst
