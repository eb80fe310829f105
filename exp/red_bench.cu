// Microbenchmark: fp32 reduction throughput into L2/HBM on sm_100a.
//   mode 0: red.global.add.v4.f32 (warp covers 512 contiguous bytes)
//   mode 1: cp.reduce.async.bulk.global.shared::cta.add.f32 from SMEM (16 KB ops)
//   mode 2: st.global.v4 (plain store, upper bound)
// Each CTA reduces a 64 KB tile per round into a target region of `region_mb`.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(128) k_red(float* dst, size_t region_floats, int rounds, int mode, int groups) {
  extern __shared__ __align__(128) float sm[];   // 32 KB staging (2 x 16 KB)
  const int t = threadIdx.x;
  for (int i = t; i < 8192; i += 128) sm[i] = 1.0f;
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  size_t tile = 16384;  // floats per 64 KB tile
  size_t ntiles = region_floats / tile;
  for (int r = 0; r < rounds; ++r) {
    size_t tidx = groups <= 0 ? ((size_t)blockIdx.x * 7919 + (size_t)r * 131) % ntiles
                            : ((size_t)r + (size_t)(blockIdx.x % groups) * (ntiles / groups)) % ntiles;
    float* base = dst + tidx * tile;
    if (mode == 0) {
#pragma unroll 4
      for (int j = 0; j < 32; ++j) {
        float* a = base + ((size_t)j * 128 + t) * 4;
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(a), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
      }
    } else if (mode == 1) {
      if (t == 0) {
        for (int c = 0; c < 4; ++c) {
          uint32_t s = (uint32_t)__cvta_generic_to_shared(sm + (c & 1) * 4096);
          asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(base + c * 4096), "r"(s), "r"(16384) : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
      }
    } else {
#pragma unroll 4
      for (int j = 0; j < 32; ++j) {
        float4* a = reinterpret_cast<float4*>(base + ((size_t)j * 128 + t) * 4);
        *a = make_float4(1.f, 1.f, 1.f, 1.f);
      }
    }
  }
  if (mode == 1 && t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  size_t region_mb = argc > 1 ? (size_t)atoi(argv[1]) : 256;
  int groups = argc > 2 ? atoi(argv[2]) : 0;
  printf("region %zu MB, groups %d (0 = scattered; g = CTAs in g lockstep groups)\n", region_mb, groups);
  size_t nf = region_mb * 1024 * 1024 / 4;
  float* d;
  cudaMalloc(&d, nf * 4);
  cudaMemset(d, 0, nf * 4);
  cudaFuncSetAttribute(k_red, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  const char* names[3] = {"red.global.add.v4.f32", "cp.reduce.async.bulk.add.f32", "st.global.v4"};
  for (int ctas_per_sm = 1; ctas_per_sm <= 2; ++ctas_per_sm)
    for (int mode = 0; mode < 3; ++mode) {
      int grid = 148 * ctas_per_sm, rounds = 400;
      k_red<<<grid, 128, 32768>>>(d, nf, 10, mode, groups);
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      k_red<<<grid, 128, 32768>>>(d, nf, rounds, mode, groups);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      double bytes = (double)grid * rounds * 65536;
      printf("%-32s ctas/SM=%d  %8.3f ms  %8.1f GB/s\n", names[mode], ctas_per_sm, ms, bytes / ms / 1e6);
    }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
