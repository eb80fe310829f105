// HBM-bound helper kernels around the LAO kernels.
//   finalize    : O = O_acc / l, lse = (m + log2 l) ln 2   (PartialAttn.finalize,
//                 local_attn.py:127-135) for rows a causal last hop did not touch
//   preprocess  : D = rowsum(dO * O) (ring.init_backward, ring.py:207), packed with
//                 lse*log2e into the backward stats workspace (padded rows -> +inf/0)
//   bwd_finalize: dQ from its fp32 accumulator; dK/dV = sum of the per-hop
//                 contributions (sim._collect, sim.py:450-471)
#pragma once
#include <cuda_bf16.h>
#include "common.cuh"

namespace burst {
namespace aux {

template <typename T>
__device__ __forceinline__ float ld_f(const T* p);
template <>
__device__ __forceinline__ float ld_f<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ld_f<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }

template <typename T>
__device__ __forceinline__ void st4(T* p, float a, float b, float c, float d);
template <>
__device__ __forceinline__ void st4<float>(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}
template <>
__device__ __forceinline__ void st4<__nv_bfloat16>(__nv_bfloat16* p, float a, float b, float c, float d) {
  __nv_bfloat162 x = __floats2bfloat162_rn(a, b), y = __floats2bfloat162_rn(c, d);
  uint2 w;
  w.x = *reinterpret_cast<uint32_t*>(&x);
  w.y = *reinterpret_cast<uint32_t*>(&y);
  *reinterpret_cast<uint2*>(p) = w;
}

// one thread per (b, h, row, 4 columns); consecutive threads = consecutive rows
// of one TL column group, so TL reads are coalesced.
template <typename T>
__global__ void finalize_kernel(int B, int H, int D, int64_t n, const float* __restrict__ o_acc,
                                const float* __restrict__ m, const float* __restrict__ l,
                                T* __restrict__ out, float* __restrict__ lse, int* flags) {
  const int64_t NT = ceil_div(n, 128);
  const int64_t total = (int64_t)B * H * NT * (D / 4) * 128;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i & 127;
    int64_t rest = i >> 7;
    const int c4 = (int)(rest % (D / 4));
    rest /= (D / 4);
    const int64_t tile = rest % NT;
    const int64_t bh = rest / NT;
    const int64_t row = tile * 128 + r;
    if (row >= n) continue;
    const float lv = l[bh * n + row], mv = m[bh * n + row];
    const float inv = lv > 0.f ? 1.f / lv : 0.f;
    const float4 o = *reinterpret_cast<const float4*>(o_acc + i * 4);
    const int64_t b = bh / H, h = bh % H;
    st4<T>(out + ((b * n + row) * H + h) * D + c4 * 4, o.x * inv, o.y * inv, o.z * inv, o.w * inv);
    if (c4 == 0) {
      lse[bh * n + row] = lv > 0.f ? (mv + log2f(lv)) * kLn2 : -INFINITY;
      if (!(lv > 0.f)) atomicOr(flags, 1);
    }
  }
}

// one warp per (b, h, padded row)
template <typename T>
__global__ void preprocess_kernel(int B, int H, int D, int64_t n, const T* __restrict__ o,
                                  const T* __restrict__ dout, const float* __restrict__ lse,
                                  float* __restrict__ stats) {
  const int64_t NT = ceil_div(n, 128);
  const int64_t rows = (int64_t)B * H * NT * 128;
  const int lane = threadIdx.x & 31;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < rows;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t bh = w / (NT * 128), row = w % (NT * 128);
    float acc = 0.f;
    if (row < n) {
      const int64_t b = bh / H, h = bh % H;
      const int64_t base = ((b * n + row) * H + h) * D;
      for (int c = lane; c < D; c += 32) acc = fmaf(ld_f<T>(dout + base + c), ld_f<T>(o + base + c), acc);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) {
      stats[w] = row < n ? lse[bh * n + row] * kLog2e : INFINITY;
      stats[rows + w] = acc;
    }
  }
}

struct Parts {
  const float* p[16];
};

template <typename T>
__global__ void bwd_finalize_kernel(int B, int H, int D, int64_t n, const float* __restrict__ dq_acc,
                                    Parts dk, Parts dv, int nparts, T* __restrict__ dq,
                                    T* __restrict__ dko, T* __restrict__ dvo) {
  const int64_t NT = ceil_div(n, 128);
  const int64_t total = (int64_t)B * H * NT * (D / 4) * 128;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i & 127;
    int64_t rest = i >> 7;
    const int c4 = (int)(rest % (D / 4));
    rest /= (D / 4);
    const int64_t tile = rest % NT;
    const int64_t bh = rest / NT;
    const int64_t row = tile * 128 + r;
    if (row >= n) continue;
    const int64_t b = bh / H, h = bh % H;
    const int64_t dst = ((b * n + row) * H + h) * D + c4 * 4;
    if (dq != nullptr) {
      const float4 a = *reinterpret_cast<const float4*>(dq_acc + i * 4);
      st4<T>(dq + dst, a.x, a.y, a.z, a.w);
    }
    float4 sk = make_float4(0.f, 0.f, 0.f, 0.f), sv = sk;
    for (int k = 0; k < nparts; ++k) {
      const float4 a = *reinterpret_cast<const float4*>(dk.p[k] + i * 4);
      const float4 c = *reinterpret_cast<const float4*>(dv.p[k] + i * 4);
      sk.x += a.x; sk.y += a.y; sk.z += a.z; sk.w += a.w;
      sv.x += c.x; sv.y += c.y; sv.z += c.z; sv.w += c.w;
    }
    if (nparts > 0) {
      st4<T>(dko + dst, sk.x, sk.y, sk.z, sk.w);
      st4<T>(dvo + dst, sv.x, sv.y, sv.z, sv.w);
    }
  }
}

// out = sum of TL parts (gradient assembly from per-hop contributions)
template <typename T>
__global__ void tl_sum_kernel(int B, int H, int D, int64_t n, Parts parts, int nparts,
                              T* __restrict__ out) {
  const int64_t NT = ceil_div(n, 128);
  const int64_t total = (int64_t)B * H * NT * (D / 4) * 128;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i & 127;
    int64_t rest = i >> 7;
    const int c4 = (int)(rest % (D / 4));
    rest /= (D / 4);
    const int64_t tile = rest % NT;
    const int64_t bh = rest / NT;
    const int64_t row = tile * 128 + r;
    if (row >= n) continue;
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = 0; k < nparts; ++k) {
      const float4 a = *reinterpret_cast<const float4*>(parts.p[k] + i * 4);
      s.x += a.x; s.y += a.y; s.z += a.z; s.w += a.w;
    }
    const int64_t b = bh / H, h = bh % H;
    st4<T>(out + ((b * n + row) * H + h) * D + c4 * 4, s.x, s.y, s.z, s.w);
  }
}

// Zero the rows of a TL contribution buffer outside [lo, hi): a hop's LAO-bwd
// writes (accumulate = 0) only the visiting key rows it covers, so a partial
// key range (K_EARLY_HALF, padded shards) leaves the rest to this kernel.
__global__ void zero_rows_outside_kernel(int B, int H, int D, int64_t n, int64_t lo, int64_t hi,
                                         float* __restrict__ a, float* __restrict__ b) {
  const int64_t NT = ceil_div(n, 128);
  const int64_t total = (int64_t)B * H * NT * (D / 4) * 128;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = (((i >> 7) / (D / 4)) % NT) * 128 + (i & 127);
    if (row >= lo && row < hi) continue;
    if (a) reinterpret_cast<float4*>(a)[i] = z;
    if (b) reinterpret_cast<float4*>(b)[i] = z;
  }
}

}  // namespace aux
}  // namespace burst
