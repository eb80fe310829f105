// Microbenchmark: TMEM read (tcgen05.ld.32x32b.x32) and write (tcgen05.st) throughput
// per SM on sm_100a, with 4, 8 or 16 warps issuing (each warp reads its lane quadrant).
// Prints bytes/clk/SM.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I paper_2403_09347_b200/csrc exp/tmem_bw.cu -o exp/tmem_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace burst;

template <bool kStore>
__global__ void __launch_bounds__(512, 1) k(int iters, int per_wait, long long* cyc, uint32_t* sink) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) ptx::tmem_alloc(&holder, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = holder;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t col = (uint32_t)((warp >> 2) * 32) & 511u;
  uint32_t r[32];
  for (int j = 0; j < 32; ++j) r[j] = threadIdx.x + j;
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int u = 0; u < per_wait; ++u) {
      const uint32_t c = (col + 128u * (uint32_t)u) & 511u;
      if (kStore)
        ptx::tmem_st32(tbase + lane_off + c, r);
      else
        ptx::tmem_ld32(tbase + lane_off + c, r);
    }
    if (kStore) {
      ptx::tmem_wait_st();
    } else {
      ptx::tmem_wait_ld();
      ptx::reg_fence(r);
      acc += r[0] ^ r[17] ^ r[31];
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[0] = acc;
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tbase, 512);
}

int main() {
  long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  cudaMalloc(&sink, 4);
  const int iters = 4096;
  for (int store = 0; store < 2; ++store)
    for (int warps : {4, 8, 16})
      for (int per : {1, 2, 4}) {
        auto kern = store ? k<true> : k<false>;
        kern<<<148, 32 * warps>>>(iters, per, cyc, sink);
        kern<<<148, 32 * warps>>>(iters, per, cyc, sink);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        long long h[148];
        cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        const double bytes = (double)iters * per * warps * 32 * 32 * 4;   // per SM
        printf("%s warps=%2d x%d per wait: %7.1f B/clk/SM  (%.0f cycles per 4 KB warp access)\n",
               store ? "tcgen05.st" : "tcgen05.ld", warps, per, bytes / mx,
               (double)mx / (iters * per) * (warps / 4.0) / (warps / 4.0));
      }
  return 0;
}
