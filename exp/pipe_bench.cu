// Microbenchmark: per-SM throughput of MUFU.EX2, F2FP (cvt.rn.bf16x2.f32) and an
// integer round-and-pack (IADD + PRMT) on sm_100a.  Prints ops/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

template <int MODE>
__global__ void __launch_bounds__(512) k(float* out, int iters, long long* cyc) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = (threadIdx.x + i) * 1e-3f;
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      if (MODE == 0) {
        float y0, y1;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y0) : "f"(a[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y1) : "f"(a[i + 1]));
        a[i] = y0 * 0.5f; a[i + 1] = y1 * 0.5f;   // keep a dependency + an FMUL each
      } else if (MODE == 1) {
        uint32_t p;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p) : "f"(a[i + 1]), "f"(a[i]));
        acc ^= p;
        a[i] += 1.0f; a[i + 1] += 1.0f;
      } else {
        uint32_t x0 = __float_as_uint(a[i]) + 0x8000u, x1 = __float_as_uint(a[i + 1]) + 0x8000u, p;
        asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(p) : "r"(x0), "r"(x1));
        acc ^= p;
        a[i] += 1.0f; a[i + 1] += 1.0f;
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
}

int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 512 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  const char* names[3] = {"MUFU.EX2 (+FMUL)", "F2FP cvt.rn.bf16x2 (+2 FADD)", "IADD+PRMT pack (+2 FADD)"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<148, 512>>>(out, iters, cyc);
      if (mode == 1) k<1><<<148, 512>>>(out, iters, cyc);
      if (mode == 2) k<2><<<148, 512>>>(out, iters, cyc);
    }
    cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double ops = (mode == 0 ? 8.0 : 4.0) * iters * 512;   // ex2 ops or packs per SM
    printf("%-32s %8.2f ops/clk/SM (%lld cycles)\n", names[mode], ops / c, c);
  }
  return 0;
}
