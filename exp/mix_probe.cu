// Probe: can one kernel mix cta_group::2 and cta_group::1 tcgen05.mma (not product code)?
// The leader issues a 2-CTA MMA (M=256) into TMEM columns [0,128) of both CTAs, then each
// CTA issues its own 1-CTA MMA (M=128, N=128) into columns [128,256); both results are
// checked.  ALLOC2=1: TMEM allocated with cta_group::2; ALLOC2=0: cta_group::1 per CTA.
//   D[M x N] = A[M x K] * B[N x K]^T, bf16 in, fp32 out, K = 64 (one 128B swizzle atom),
//   M = 256 (128 rows per CTA) or M = 128 (64 rows per CTA, "2x2" TMEM layout), N = 128.
// Each CTA TMA-loads its half of A (M/2 rows) and its half of B (N/2 rows) with the
// .cta_group::2 form signalling the LEADER's mbarrier; the leader issues the MMAs and a
// multicast commit; each CTA reads its own TMEM and writes its D rows.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cmath>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cta_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

#ifndef ALLOC2
#define ALLOC2 1
#endif
template <int M>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
probe(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
      const __grid_constant__ CUtensorMap tBfull, float* D) {
  __shared__ __align__(1024) uint8_t sA[128 * 128];   // up to 128 rows x 64 bf16
  __shared__ __align__(1024) uint8_t sB[64 * 128];    // 64 rows x 64 bf16
  __shared__ __align__(1024) uint8_t sBf[128 * 128];  // all 128 rows of B (1-CTA MMA)
  __shared__ __align__(8) uint64_t full, done, full1, done1;
  __shared__ uint32_t holder;
  const uint32_t c = cta_rank();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int MH = M / 2;   // rows of A / D per CTA
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&done)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full1)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&done1)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
#if ALLOC2
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
#else
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
#endif
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = holder;
  // leader's barrier in the cluster window: clear the peer bit (bit 24)
  const uint32_t full_leader = su32(&full) & 0xFEFFFFFFu;
  if (threadIdx.x == 0) {
    if (c == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full)),
                   "r"((uint32_t)(2 * (MH * 128 + 64 * 128))) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(su32(sA)), "l"((uint64_t)&tA), "r"(full_leader),
        "r"(0), "r"((int)(c * MH)) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(su32(sB)), "l"((uint64_t)&tB), "r"(full_leader),
        "r"(0), "r"((int)(c * 64)) : "memory");
  }
  if (c == 0 && threadIdx.x == 32) {
    uint32_t ok = 0;
    while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(su32(&full)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int kk = 0; kk < 4; ++kk) {
      uint64_t a = sdesc(su32(sA) + kk * 32, 0, 1024), b = sdesc(su32(sB) + kk * 32, 0, 1024);
      asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;}"
                   ::"r"(tbase), "l"(a), "l"(b), "r"(idesc(M, 128)), "r"((uint32_t)(kk > 0)));
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(su32(&done)), "h"((uint16_t)3) : "memory");
  }
  // every CTA: wait for the 2-CTA MMA
  {
    uint32_t ok = 0;
    while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(su32(&done)) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // then each CTA: its own 1-CTA MMA D1[128 x 128] = A_c[128 x 64] * Bfull[128 x 64]^T into
  // columns [128, 256) (A_c = this CTA's 128 rows of A, already in sA for M=256)
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full1)),
                 "r"((uint32_t)(128 * 128)) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(su32(sBf)), "l"((uint64_t)&tBfull), "r"(su32(&full1)),
        "r"(0), "r"(0) : "memory");
    uint32_t ok = 0;
    while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(su32(&full1)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int kk = 0; kk < 4; ++kk) {
      uint64_t a = sdesc(su32(sA) + kk * 32, 0, 1024), b = sdesc(su32(sBf) + kk * 32, 0, 1024);
      asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                   ::"r"(tbase + 128), "l"(a), "l"(b), "r"(idesc(128, 128)), "r"((uint32_t)(kk > 0)));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 ::"r"(su32(&done1)) : "memory");
  }
  {
    uint32_t ok = 0;
    while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(su32(&done1)) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // thread t reads TMEM lane t, 128 columns
  uint32_t r[32];
  for (int cc = 0; cc < 8; ++cc) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(tbase + ((uint32_t)(warp * 32) << 16) + cc * 32));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    // raw dump: D_raw[c][lane][col]
    for (int i = 0; i < 32; ++i) D[((size_t)c * 128 + threadIdx.x) * 256 + cc * 32 + i] = __uint_as_float(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
#if ALLOC2
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tbase));
#else
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
#endif
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return (PFN_cuTensorMapEncodeTiled_v12000)p;
}
static void tmap(CUtensorMap* t, void* base, int rows, int box_rows) {
  cuuint64_t dims[2] = {64, (cuuint64_t)rows}, str[1] = {128};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows}, es[2] = {1, 1};
  CUresult r = enc()(t, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) printf("tmap err %d\n", (int)r);
}

void run() {
  constexpr int M = 256;
  std::vector<__nv_bfloat16> hA(M * 64), hB(128 * 64);
  std::vector<float> fA(M * 64), fB(128 * 64);
  for (int i = 0; i < M * 64; ++i) { float x = (float)((i * 37 % 17) - 8) / 8.f; hA[i] = __float2bfloat16(x); fA[i] = __bfloat162float(hA[i]); }
  for (int i = 0; i < 128 * 64; ++i) { float x = (float)((i * 53 % 13) - 6) / 8.f; hB[i] = __float2bfloat16(x); fB[i] = __bfloat162float(hB[i]); }
  __nv_bfloat16 *dA, *dB; float* dD;
  cudaMalloc(&dA, M * 64 * 2); cudaMalloc(&dB, 128 * 64 * 2); cudaMalloc(&dD, 2 * 128 * 256 * 4);
  cudaMemcpy(dA, hA.data(), M * 64 * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), 128 * 64 * 2, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, 2 * 128 * 256 * 4);
  CUtensorMap tA, tB, tBf;
  tmap(&tA, dA, M, M / 2);
  tmap(&tB, dB, 128, 64);
  tmap(&tBf, dB, 128, 128);
  probe<M><<<2, 128>>>(tA, tB, tBf, dD);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> raw(2 * 128 * 256);
  cudaMemcpy(raw.data(), dD, raw.size() * 4, cudaMemcpyDeviceToHost);
  auto ref = [&](int m, int n) { float s = 0; for (int k = 0; k < 64; ++k) s += fA[m * 64 + k] * fB[n * 64 + k]; return s; };
  double e2 = 0, e1 = 0;
  for (int c = 0; c < 2; ++c) for (int l = 0; l < 128; ++l) for (int n = 0; n < 128; ++n) {
    e2 = fmax(e2, fabs(raw[((size_t)c * 128 + l) * 256 + n] - ref(c * 128 + l, n)));
    e1 = fmax(e1, fabs(raw[((size_t)c * 128 + l) * 256 + 128 + n] - ref(c * 128 + l, n)));
  }
  printf("ALLOC2=%d: %s; 2-CTA MMA max err %.3e; 1-CTA MMA (same kernel) max err %.3e\n", ALLOC2,
         cudaGetErrorString(e), e2, e1);
}

int main() {
  run();
  return 0;
}
