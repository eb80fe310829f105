// HBM-bound helper kernels around the LAO kernels.
//   preprocess  : D = rowsum(dO * O) (ring.init_backward, ring.py:207), packed with
//                 lse*log2e into the backward stats workspace (padded rows -> +inf/0)
//   tl_rows     : TL workspace -> row-major output: dQ from its fp32 accumulator,
//                 dK/dV = sum of the per-hop contributions (sim._collect,
//                 sim.py:450-471), or the forward finalize O = O_acc / l with lse
//                 (PartialAttn.finalize, local_attn.py:127-135)
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
__device__ __forceinline__ void ld4(const T* p, float* x);
template <>
__device__ __forceinline__ void ld4<float>(const float* p, float* x) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
}
template <>
__device__ __forceinline__ void ld4<__nv_bfloat16>(const __nv_bfloat16* p, float* x) {
  const uint2 v = *reinterpret_cast<const uint2*>(p);
  const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&v.x);
  const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&v.y);
  x[0] = __low2float(a); x[1] = __high2float(a); x[2] = __low2float(b); x[3] = __high2float(b);
}

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

// one warp per (b, h, padded row)
template <typename T>
__global__ void preprocess_kernel(int B, int H, int D, int64_t n, const T* __restrict__ o,
                                  const T* __restrict__ dout, const float* __restrict__ lse,
                                  float* __restrict__ stats, bool vec) {
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
      if (vec) {
        // 4 consecutive elements per lane (8 B bf16 / 16 B f32 loads)
        for (int c = lane * 4; c < D; c += 128) {
          float x[4], y[4];
          ld4<T>(dout + base + c, x);
          ld4<T>(o + base + c, y);
#pragma unroll
          for (int e = 0; e < 4; ++e) acc = fmaf(x[e], y[e], acc);
        }
      } else {
        for (int c = lane; c < D; c += 32) acc = fmaf(ld_f<T>(dout + base + c), ld_f<T>(o + base + c), acc);
      }
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

// TL workspace -> row-major [B, n, H, D] output through a shared-memory transpose.
// One block per (b*h, 128-row tile, 32-column group): the TL reads are one float4
// per thread along the tile's rows (coalesced), the output writes are 64-128 B
// runs along each row (a per-thread row-major store would touch one 8-16 B piece
// of a different row per thread, 4x write amplification).
//   kFinal = false: out = sum of the TL parts (dQ from its accumulator, dK/dV from
//                   the per-hop contributions, sim._collect sim.py:450-471)
//   kFinal = true : out = O_acc / l and lse = (m + log2 l) ln 2 (PartialAttn.finalize,
//                   local_attn.py:127-135), parts.p[0] = O_acc
template <typename T, bool kFinal>
__global__ void __launch_bounds__(256) tl_rows_kernel(int H, int D, int64_t n, Parts parts, int nparts,
                                                      T* __restrict__ out, const float* __restrict__ m,
                                                      const float* __restrict__ l, float* __restrict__ lse,
                                                      int* flags) {
  __shared__ float4 s4[128 * 9];   // 128 rows x (8 float4 + 1 pad): conflict-free both ways
  const int cw = D < 32 ? D : 32, nc4 = cw / 4, ng = D / cw;
  const int64_t NT = ceil_div(n, 128);
  int64_t blk = blockIdx.x;
  const int cg = (int)(blk % ng);
  blk /= ng;
  const int64_t tile = blk % NT, bh = blk / NT;
  const int64_t base = ((bh * NT + tile) * (D / 4) + cg * nc4) * 128;   // float4 index
  // up to 4 float4 per thread (nc4 * 128 <= 1024): all loads of a part in flight at once
  float4 a[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int k = threadIdx.x + 256 * u;
    if (k < nc4 * 128) a[u] = reinterpret_cast<const float4*>(parts.p[0])[base + k];
  }
  for (int j = 1; j < nparts; ++j) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = threadIdx.x + 256 * u;
      if (k < nc4 * 128) {
        const float4 c = reinterpret_cast<const float4*>(parts.p[j])[base + k];
        a[u].x += c.x; a[u].y += c.y; a[u].z += c.z; a[u].w += c.w;
      }
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int k = threadIdx.x + 256 * u;   // = c4 * 128 + r
    if (k < nc4 * 128) s4[(k & 127) * 9 + (k >> 7)] = a[u];
  }
  __syncthreads();
  const int64_t b = bh / H, h = bh % H;
  float nf = 0.f;   // NaN iff an output value is non-finite (x * 0 = NaN for inf / NaN)
  for (int k = threadIdx.x; k < nc4 * 128; k += 256) {
    const int r = k / nc4, g = k % nc4;
    const int64_t row = tile * 128 + r;
    if (row >= n) continue;
    float4 v = s4[r * 9 + g];
    if (kFinal) {
      const float lv = l[bh * n + row];
      const float inv = lv > 0.f ? 1.f / lv : 0.f;
      v.x *= inv; v.y *= inv; v.z *= inv; v.w *= inv;
      if (cg == 0 && g == 0) {
        const float ls = lv > 0.f ? (m[bh * n + row] + log2f(lv)) * kLn2 : -INFINITY;
        lse[bh * n + row] = ls;
        if (lv == 0.f) atomicOr(flags, 1);                // MaskError
        else nf = fmaf(ls, 0.f, nf);
      }
    }
    nf = fmaf(v.x, 0.f, fmaf(v.y, 0.f, fmaf(v.z, 0.f, fmaf(v.w, 0.f, nf))));
    st4<T>(out + ((b * n + row) * H + h) * D + cg * cw + g * 4, v.x, v.y, v.z, v.w);
  }
  // NonFiniteError (bit 1): every public output is checked once (linalg.py:253-255)
  if (__syncthreads_or(!(fabsf(nf) <= 3.0e38f)) && threadIdx.x == 0) atomicOr(flags, 2);
}

// acc += part over a TL workspace (float4 grid-stride): folds a dK/dV (or dQ)
// contribution into the home accumulator as soon as its exchange has landed, so a
// rank holds O(1) contribution buffers whatever the ring size (ring.py:239-241
// accumulates in place the same way).
__global__ void tl_accumulate_kernel(int64_t n4, float4* __restrict__ acc,
                                     const float4* __restrict__ part) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = acc[i], c = part[i];
    acc[i] = make_float4(a.x + c.x, a.y + c.y, a.z + c.z, a.w + c.w);
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
