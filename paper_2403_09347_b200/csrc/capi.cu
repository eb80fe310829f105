// C ABI (include/burst_b200.h): argument validation, TMA tensor maps, launch
// configuration, error mapping onto the reference taxonomy (errors.py:4-33).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <set>
#include <utility>
#include <string>

#include "../../include/burst_b200.h"
#include "aux_kernels.cuh"
#include "lao_bwd4_sm100.cuh"
#include "lao_dq_sm100.cuh"
#include "lao_fwd_sm100.cuh"
#include "simt_f32.cuh"

using namespace burst;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(x)                                                                  \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) return fail(BURST_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define CHECK_LAUNCH()                                                               \
  do {                                                                               \
    cudaError_t e_ = cudaGetLastError();                                             \
    if (e_ != cudaSuccess) return fail(BURST_E_CUDA, std::string("launch: ") + cudaGetErrorString(e_)); \
  } while (0)

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 4-D map over a [B, n, H, D] bf16 tensor; box = 64 columns x 1 head x 128 rows.
int make_tmap(CUtensorMap* tm, const void* base, int64_t n, int H, int D, int B,
              int box_rows = 128) {
  auto fn = encode_fn();
  if (!fn) return fail(BURST_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0)
    return fail(BURST_E_SHAPE, "tensor base must be 16-byte aligned");
  cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)H, (cuuint64_t)n, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)D * 2, (cuuint64_t)H * D * 2, (cuuint64_t)n * H * D * 2};
  cuuint32_t box[4] = {64, 1, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(BURST_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return BURST_OK;
}

// f32 TL workspace [B*H][NT][D/4][128][4] viewed as a 3-D tensor [G][128][4]
// (G = B*H*NT*D/4 column groups) for TMA tensor reductions of 8-group x 64-row boxes.
int make_tmap_tl(CUtensorMap* tm, const float* base, int64_t n, int H, int D, int B) {
  auto fn = encode_fn();
  if (!fn) return fail(BURST_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int64_t G = (int64_t)B * H * ceil_div(n, 128) * (D / 4);
  if (G > INT32_MAX) return fail(BURST_E_SHAPE, "workspace too large for TMA coordinates");
  cuuint64_t dims[3] = {4, 128, (cuuint64_t)G};
  cuuint64_t strides[2] = {16, 2048};
  cuuint32_t box[3] = {4, 64, 8};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(BURST_E_CUDA, "cuTensorMapEncodeTiled (TL) failed: " + std::to_string((int)r));
  return BURST_OK;
}

int* device_flags() {
  static int* flags[64] = {nullptr};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (!flags[dev]) {
    if (cudaMalloc(&flags[dev], sizeof(int)) != cudaSuccess) return nullptr;
    cudaMemset(flags[dev], 0, sizeof(int));
  }
  return flags[dev];
}

#ifdef BURST_LIFE
unsigned long long* life_buffer() {
  static unsigned long long* buf = nullptr;
  if (!buf) { cudaMalloc(&buf, 65536 * 16 * sizeof(unsigned long long)); cudaMemset(buf, 0, 65536 * 16 * sizeof(unsigned long long)); }
  return buf;
}
#endif
#ifdef BURST_TRACE
long long* trace_buffer() {
  static long long* buf = nullptr;
  if (!buf) { cudaMalloc(&buf, 32 * 64 * sizeof(long long)); cudaMemset(buf, 0, 32 * 64 * sizeof(long long)); }
  return buf;
}
#endif

bool valid_map(const burst_posmap& m) { return m.seg_len >= 0 && m.pos0 + m.seg_len <= m.pos1; }

int check_hop(const burst_hop* h) {
  if (!h) return fail(BURST_E_SHAPE, "hop descriptor is null");
  if (h->batch < 1 || h->heads < 1) return fail(BURST_E_SHAPE, "batch and heads must be positive");
  if (h->n_q < 0 || h->n_k < 0 || h->q_begin < 0 || h->k_begin < 0 || h->q_len < 0 || h->k_len < 0 ||
      h->q_begin + h->q_len > h->n_q || h->k_begin + h->k_len > h->n_k)
    return fail(BURST_E_SHAPE, "hop row ranges exceed the q/k extents");
  if (!(h->softmax_scale > 0.f)) return fail(BURST_E_SHAPE, "softmax_scale must be finite and positive");
  if (h->n_q > INT32_MAX || h->n_k > INT32_MAX) return fail(BURST_E_SHAPE, "sequence too long for TMA coordinates");
  if (h->grid_skip && (h->grid_nqb < 1 || h->grid_nkb < 1 || h->grid_qcell < 1 || h->grid_kcell < 1))
    return fail(BURST_E_SHAPE, "grid mask needs positive block counts and cell extents");
  if (h->grid_skip && (!valid_map(h->q_map) || !valid_map(h->k_map)))
    return fail(BURST_E_SHAPE, "position maps must be monotone (pos0 + seg_len <= pos1)");
  if (h->causal && (!valid_map(h->q_map) || !valid_map(h->k_map)))
    return fail(BURST_E_SHAPE, "position maps must be monotone (pos0 + seg_len <= pos1)");
  if (h->dtype == BURST_DTYPE_BF16) {
    if (h->head_dim != 64 && h->head_dim != 128)
      return fail(BURST_E_UNSUPPORTED, "bf16 path supports head_dim 64 or 128");
    if ((h->q_begin % 8) || (h->k_begin % 8))
      return fail(BURST_E_SHAPE, "bf16 path needs q_begin/k_begin multiples of 8");
  } else if (h->dtype == BURST_DTYPE_F32) {
    if (h->head_dim != 16 && h->head_dim != 32 && h->head_dim != 64)
      return fail(BURST_E_UNSUPPORTED, "f32 path supports head_dim 16, 32 or 64");
  } else {
    return fail(BURST_E_UNSUPPORTED, "dtype must be BURST_DTYPE_BF16 or BURST_DTYPE_F32");
  }
  return BURST_OK;
}

// The dynamic-SMEM opt-in is a per-device (per-context) function attribute: set it
// once for every (kernel, device) pair this process launches on.
template <typename K>
int set_smem(K kernel, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  const auto key = std::make_pair(reinterpret_cast<const void*>(kernel), dev);
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(key)) return BURST_OK;
  CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.insert(key);
  return BURST_OK;
}

int* flags_of(const burst_hop* h) { return h->flags ? h->flags : device_flags(); }
int* flags_or_default(int32_t* f) { return f ? f : device_flags(); }

// Default backward: consecutive key tiles in clusters of this many CTAs sharing Q/dO
// loads (lao_bwd4 kCl; 1 = no clusters).
#ifndef BURST_BWD_CLUSTER
#define BURST_BWD_CLUSTER 2
#endif

#ifndef BURST_FWD_PAIRS
#define BURST_FWD_PAIRS 1
#endif

// Launch `kernel` as `cl`-CTA clusters along x (grid.x rounded up to a multiple of cl).
template <typename K, typename P>
int launch_pair(K kernel, dim3 grid, int threads, int smem, cudaStream_t st, const P& p,
                int cl = 2) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((grid.x + cl - 1) / cl * cl, grid.y, grid.z);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kernel, p));
  return BURST_OK;
}

int grid_for(int64_t work, int block) {
  int64_t g = (work + block - 1) / block;
  if (g > 148 * 32) g = 148 * 32;
  return (int)(g < 1 ? 1 : g);
}

template <int D>
int launch_fwd_bf16(const burst_hop* h, const void* q, const void* k, const void* v, float* o_acc,
                    float* m, float* l, void* o_out, float* lse, int first, int fin, cudaStream_t st) {
  fwd::Params p;
  memset(&p, 0, sizeof(p));
  int rc;
  if ((rc = make_tmap(&p.tm_q, q, h->n_q, h->heads, D, h->batch))) return rc;
  if ((rc = make_tmap(&p.tm_k, k, h->n_k, h->heads, D, h->batch))) return rc;
  if ((rc = make_tmap(&p.tm_v, v, h->n_k, h->heads, D, h->batch))) return rc;
  p.o_acc = o_acc; p.m_run = m; p.l_run = l; p.o_out = o_out; p.lse_out = lse;
  p.flags = flags_of(h);
  p.hop = *h;
  p.scale_log2 = h->softmax_scale * kLog2e;
  p.first_hop = first; p.finalize = fin;
#ifdef BURST_TRACE
  p.trace = trace_buffer();
#endif
  dim3 grid((unsigned)ceil_div(h->q_len, 2 * fwd::BM), h->heads, h->batch);
  const bool general = h->grid_skip || h->key_order;
  constexpr bool kPairs = (D == 128) && BURST_FWD_PAIRS;
  if constexpr (kPairs) {
    // query-block pairs as 2-CTA clusters sharing K/V (TMA multicast); an odd block count
    // gets one row-less CTA that only consumes its half of the shared stages
    auto kernel = general ? fwd::lao_fwd_kernel<D, true, true> : fwd::lao_fwd_kernel<D, false, true>;
    if ((rc = set_smem(kernel, fwd::Cfg<D>::kSmemBytes))) return rc;
    rc = launch_pair(kernel, grid, fwd::kThreads, fwd::Cfg<D>::kSmemBytes, st, p);
    if (rc) return rc;
  } else {
    auto kernel = general ? fwd::lao_fwd_kernel<D, true> : fwd::lao_fwd_kernel<D, false>;
    if ((rc = set_smem(kernel, fwd::Cfg<D>::kSmemBytes))) return rc;
    kernel<<<grid, fwd::kThreads, fwd::Cfg<D>::kSmemBytes, st>>>(p);
  }
  CHECK_LAUNCH();
  return BURST_OK;
}

template <int D>
int launch_fwd_f32(const burst_hop* h, const void* q, const void* k, const void* v, float* o_acc,
                   float* m, float* l, void* o_out, float* lse, int first, int fin, cudaStream_t st) {
  simt::FwdParams p;
  p.q = (const float*)q; p.k = (const float*)k; p.v = (const float*)v;
  p.o_acc = o_acc; p.m_run = m; p.l_run = l; p.o_out = (float*)o_out; p.lse_out = lse;
  p.flags = flags_of(h);
  p.hop = *h;
  p.scale_log2 = h->softmax_scale * kLog2e;
  p.first_hop = first; p.finalize = fin;
  dim3 grid((unsigned)ceil_div(h->q_len, simt::kRows), h->heads, h->batch);
  simt::simt_fwd_kernel<D><<<grid, simt::kRows, 0, st>>>(p);
  CHECK_LAUNCH();
  return BURST_OK;
}

// Deterministic dQ (query-stationary, one writer per dQ row; lao_dq_sm100.cuh).
template <int D>
int launch_dq_bf16(const burst_hop* h, const void* q, const void* k, const void* v, const void* dout,
                   const float* stats, float* dq_acc, cudaStream_t st) {
  if (h->q_len <= 0) return BURST_OK;   // no query rows: no dQ contribution
  bdq::Params p;
  memset(&p, 0, sizeof(p));
  int rc;
  if ((rc = make_tmap(&p.tm_q, q, h->n_q, h->heads, D, h->batch))) return rc;
  if ((rc = make_tmap(&p.tm_do, dout, h->n_q, h->heads, D, h->batch))) return rc;
  if ((rc = make_tmap(&p.tm_k, k, h->n_k, h->heads, D, h->batch))) return rc;
  if ((rc = make_tmap(&p.tm_v, v, h->n_k, h->heads, D, h->batch))) return rc;
  p.stats = stats;
  p.dq_acc = dq_acc;
  p.hop = *h;
  p.hop.flags = flags_of(h);
  p.scale_log2 = h->softmax_scale * kLog2e;
  p.scale = h->softmax_scale;
  dim3 grid((unsigned)ceil_div(h->q_len, bdq::BM), h->heads, h->batch);
  auto go = [&](auto kernel) -> int {
    if (int e = set_smem(kernel, bdq::Cfg<D>::kSmemBytes)) return e;
    kernel<<<grid, bdq::kThreads, bdq::Cfg<D>::kSmemBytes, st>>>(p);
    return BURST_OK;
  };
  rc = h->grid_skip ? go(bdq::lao_dq_kernel<D, true>) : go(bdq::lao_dq_kernel<D, false>);
  if (rc) return rc;
  CHECK_LAUNCH();
  return BURST_OK;
}

template <int D>
int launch_bwd4_bf16(const burst_hop* h, const void* q, const void* k, const void* v, const void* dout,
                     const float* stats, float* dq_acc, float* dk, float* dv, int acc, cudaStream_t st) {
  bwd4::Params p;
  memset(&p, 0, sizeof(p));
  int rc;
  if ((rc = make_tmap(&p.tm_q, q, h->n_q, h->heads, D, h->batch))) return rc;
  if ((rc = make_tmap(&p.tm_do, dout, h->n_q, h->heads, D, h->batch))) return rc;
  if ((rc = make_tmap(&p.tm_k, k, h->n_k, h->heads, D, h->batch))) return rc;
  if ((rc = make_tmap(&p.tm_v, v, h->n_k, h->heads, D, h->batch))) return rc;
  p.stats = stats; p.dq_acc = dq_acc; p.dk_acc = dk; p.dv_acc = dv;
  p.hop = *h;
  p.hop.flags = flags_of(h);
  p.scale_log2 = h->softmax_scale * kLog2e;
  p.scale = h->softmax_scale;
  p.accumulate = acc;
#ifdef BURST_TRACE
  p.trace = trace_buffer();
#endif
#ifdef BURST_LIFE
  p.life = life_buffer();
#endif
  dim3 grid((unsigned)ceil_div(h->k_len, bwd4::BN), h->heads, h->batch);
  auto go = [&](auto kernel) -> int {
    if (int e = set_smem(kernel, bwd4::Cfg<D>::kSmemBytes)) return e;
    kernel<<<grid, bwd4::kThreads, bwd4::Cfg<D>::kSmemBytes, st>>>(p);
    return BURST_OK;
  };
  // key-tile pairs as 2-CTA clusters sharing Q/dO loads (TMA multicast); an odd tile
  // count gets one key-less CTA that only consumes its half of the shared stages
  auto go_pair = [&](auto kernel) -> int {
    if (int e = set_smem(kernel, bwd4::Cfg<D>::kSmemBytes)) return e;
    return launch_pair(kernel, grid, bwd4::kThreads, bwd4::Cfg<D>::kSmemBytes, st, p,
                       D == 128 ? BURST_BWD_CLUSTER : 1);
  };
  constexpr int kCl = D == 128 ? BURST_BWD_CLUSTER : 1;
  if (kCl == 4) {
    if ((rc = make_tmap(&p.tm_q64, q, h->n_q, h->heads, D, h->batch, 64))) return rc;
    if ((rc = make_tmap(&p.tm_do64, dout, h->n_q, h->heads, D, h->batch, 64))) return rc;
  }
  if constexpr (kCl > 1) {
    if (h->dq_order)   // deterministic: dK/dV only (dQ from lao_dq below)
      rc = h->grid_skip ? go_pair(bwd4::lao_bwd4_kernel<D, true, true, kCl>)
                        : go_pair(bwd4::lao_bwd4_kernel<D, false, true, kCl>);
    else
      rc = h->grid_skip ? go_pair(bwd4::lao_bwd4_kernel<D, true, false, kCl>)
                        : go_pair(bwd4::lao_bwd4_kernel<D, false, false, kCl>);
  } else if (h->dq_order) {
    rc = h->grid_skip ? go(bwd4::lao_bwd4_kernel<D, true, true>) : go(bwd4::lao_bwd4_kernel<D, false, true>);
  } else {
    rc = h->grid_skip ? go(bwd4::lao_bwd4_kernel<D, true, false>) : go(bwd4::lao_bwd4_kernel<D, false, false>);
  }
  if (rc) return rc;
  CHECK_LAUNCH();
  if (h->dq_order) return launch_dq_bf16<D>(h, q, k, v, dout, stats, dq_acc, st);
  return BURST_OK;
}

template <int D>
int launch_bwd_f32(const burst_hop* h, const void* q, const void* k, const void* v, const void* dout,
                   const float* stats, float* dq_acc, float* dk, float* dv, int acc, cudaStream_t st) {
  simt::BwdParams p;
  p.q = (const float*)q; p.k = (const float*)k; p.v = (const float*)v; p.dout = (const float*)dout;
  p.stats = stats; p.dq_acc = dq_acc; p.dk_acc = dk; p.dv_acc = dv;
  p.hop = *h;
  p.hop.flags = flags_of(h);
  p.scale_log2 = h->softmax_scale * kLog2e;
  p.scale = h->softmax_scale;
  p.accumulate = acc;
  const int smem = 2 * simt::kRows * (D + 1) * 4;
  if (int rc = set_smem(simt::simt_bwd_dkv_kernel<D>, smem)) return rc;
  if (h->q_len > 0) {
    dim3 g1((unsigned)ceil_div(h->q_len, simt::kRows), h->heads, h->batch);
    simt::simt_bwd_dq_kernel<D><<<g1, simt::kRows, 0, st>>>(p);
    CHECK_LAUNCH();
  }
  dim3 g2((unsigned)ceil_div(h->k_len, simt::kRows), h->heads, h->batch);
  simt::simt_bwd_dkv_kernel<D><<<g2, simt::kRows, smem, st>>>(p);
  CHECK_LAUNCH();
  return BURST_OK;
}

int check_dims(int dtype, int B, int H, int D, int64_t n) {
  if (B < 1 || H < 1 || n < 0) return fail(BURST_E_SHAPE, "batch/heads must be positive, n >= 0");
  if (dtype == BURST_DTYPE_BF16 && D != 64 && D != 128)
    return fail(BURST_E_UNSUPPORTED, "bf16 path supports head_dim 64 or 128");
  if (dtype == BURST_DTYPE_F32 && D != 16 && D != 32 && D != 64)
    return fail(BURST_E_UNSUPPORTED, "f32 path supports head_dim 16, 32 or 64");
  if (dtype != BURST_DTYPE_BF16 && dtype != BURST_DTYPE_F32) return fail(BURST_E_UNSUPPORTED, "bad dtype");
  return BURST_OK;
}

}  // namespace

#ifdef BURST_LIFE
extern "C" __attribute__((visibility("default"))) int burst_exp_life_read(unsigned long long* host) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpy(host, life_buffer(), 65536 * 16 * sizeof(unsigned long long),
                         cudaMemcpyDeviceToHost);
}
#endif
#ifdef BURST_TRACE
extern "C" __attribute__((visibility("default"))) int burst_exp_trace_read(long long* host) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpy(host, trace_buffer(), 32 * 64 * sizeof(long long), cudaMemcpyDeviceToHost);
}
#endif

int burst_internal_fail(int code, const std::string& msg) { return fail(code, msg); }

extern "C" {

int burst_version(void) { return 1; }

const char* burst_last_error(void) { return g_err.c_str(); }

size_t burst_workspace_floats(int batch, int heads, int head_dim, int64_t n) {
  return (size_t)batch * heads * (size_t)ceil_div(n, 128) * 128 * head_dim;
}

int burst_lao_fwd(const burst_hop* hop, const void* q, const void* k, const void* v, float* o_acc,
                  float* m, float* l, void* o_out, float* lse_out, int first_hop, int finalize,
                  void* stream) {
  int rc = check_hop(hop);
  if (rc) return rc;
  if (!finalize && (!o_acc || !m || !l)) return fail(BURST_E_SHAPE, "running state pointers are null");
  if (finalize && (!o_out || !lse_out)) return fail(BURST_E_SHAPE, "output pointers are null");
  if (!first_hop && (!o_acc || !m || !l))
    return fail(BURST_E_ORDER, "non-first hop needs the running state (init_forward first)");
  if (hop->q_len == 0) return BURST_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (hop->dtype == BURST_DTYPE_BF16) {
    if (hop->head_dim == 128)
      return launch_fwd_bf16<128>(hop, q, k, v, o_acc, m, l, o_out, lse_out, first_hop, finalize, st);
    return launch_fwd_bf16<64>(hop, q, k, v, o_acc, m, l, o_out, lse_out, first_hop, finalize, st);
  }
  switch (hop->head_dim) {
    case 16: return launch_fwd_f32<16>(hop, q, k, v, o_acc, m, l, o_out, lse_out, first_hop, finalize, st);
    case 32: return launch_fwd_f32<32>(hop, q, k, v, o_acc, m, l, o_out, lse_out, first_hop, finalize, st);
    default: return launch_fwd_f32<64>(hop, q, k, v, o_acc, m, l, o_out, lse_out, first_hop, finalize, st);
  }
}

// TL workspace -> row-major output (aux::tl_rows_kernel), one block per
// (b*h, 128-row tile, 32-column group).
static void launch_tl_rows(int dtype, bool final_, int batch, int heads, int head_dim, int64_t n,
                           const aux::Parts& parts, int nparts, void* out, const float* m,
                           const float* l, float* lse, int* flags, cudaStream_t st) {
  const int cw = head_dim < 32 ? head_dim : 32;
  const int64_t blocks = (int64_t)batch * heads * ceil_div(n, 128) * (head_dim / cw);
  if (dtype == BURST_DTYPE_BF16) {
    if (final_)
      aux::tl_rows_kernel<__nv_bfloat16, true><<<(unsigned)blocks, 256, 0, st>>>(
          heads, head_dim, n, parts, nparts, (__nv_bfloat16*)out, m, l, lse, flags);
    else
      aux::tl_rows_kernel<__nv_bfloat16, false><<<(unsigned)blocks, 256, 0, st>>>(
          heads, head_dim, n, parts, nparts, (__nv_bfloat16*)out, m, l, lse, flags);
  } else {
    if (final_)
      aux::tl_rows_kernel<float, true><<<(unsigned)blocks, 256, 0, st>>>(
          heads, head_dim, n, parts, nparts, (float*)out, m, l, lse, flags);
    else
      aux::tl_rows_kernel<float, false><<<(unsigned)blocks, 256, 0, st>>>(
          heads, head_dim, n, parts, nparts, (float*)out, m, l, lse, flags);
  }
}

int burst_fwd_finalize(int dtype, int batch, int heads, int head_dim, int64_t n, const float* o_acc,
                       const float* m, const float* l, void* o_out, float* lse_out, int32_t* flags,
                       void* stream) {
  int rc = check_dims(dtype, batch, heads, head_dim, n);
  if (rc) return rc;
  if (n == 0) return BURST_OK;
  aux::Parts pp{};
  pp.p[0] = o_acc;
  launch_tl_rows(dtype, true, batch, heads, head_dim, n, pp, 1, o_out, m, l, lse_out,
                 flags_or_default(flags), (cudaStream_t)stream);
  CHECK_LAUNCH();
  return BURST_OK;
}

int burst_bwd_preprocess(int dtype, int batch, int heads, int head_dim, int64_t n, const void* o,
                         const void* dout, const float* lse, float* stats, float* dq_acc, void* stream) {
  int rc = check_dims(dtype, batch, heads, head_dim, n);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t ws = burst_workspace_floats(batch, heads, head_dim, n);
  if (dq_acc) CUDA_TRY(cudaMemsetAsync(dq_acc, 0, ws * sizeof(float), st));
  if (n == 0) return BURST_OK;
  const int64_t rows = (int64_t)batch * heads * ceil_div(n, 128) * 128;
  // 4-element vector loads when both tensors are aligned to 4 elements
  const uintptr_t align = dtype == BURST_DTYPE_BF16 ? 8 : 16;
  const bool vec = (((uintptr_t)o | (uintptr_t)dout) % align) == 0;
  if (dtype == BURST_DTYPE_BF16)
    aux::preprocess_kernel<__nv_bfloat16><<<grid_for(rows * 32, 256), 256, 0, st>>>(
        batch, heads, head_dim, n, (const __nv_bfloat16*)o, (const __nv_bfloat16*)dout, lse, stats, vec);
  else
    aux::preprocess_kernel<float><<<grid_for(rows * 32, 256), 256, 0, st>>>(
        batch, heads, head_dim, n, (const float*)o, (const float*)dout, lse, stats, vec);
  CHECK_LAUNCH();
  return BURST_OK;
}

int burst_lao_bwd(const burst_hop* hop, const void* q, const void* k, const void* v, const void* dout,
                  const float* stats, float* dq_acc, float* dk_acc, float* dv_acc, int accumulate,
                  void* stream) {
  int rc = check_hop(hop);
  if (rc) return rc;
  if (!stats) return fail(BURST_E_ORDER, "backward needs the preprocess stats (forward lse, D)");
  cudaStream_t st = (cudaStream_t)stream;
  if (!accumulate && (hop->k_begin > 0 || hop->k_begin + hop->k_len < hop->n_k)) {
    // accumulate = 0 defines the whole contribution buffer: rows the hop does not
    // cover are zero (their sum in burst_bwd_finalize must not see stale memory)
    const int64_t work = (int64_t)burst_workspace_floats(hop->batch, hop->heads, hop->head_dim,
                                                         hop->n_k) / 4;
    aux::zero_rows_outside_kernel<<<grid_for(work, 256), 256, 0, st>>>(
        hop->batch, hop->heads, hop->head_dim, hop->n_k, hop->k_begin, hop->k_begin + hop->k_len,
        dk_acc, dv_acc);
    CHECK_LAUNCH();
  }
  if (hop->k_len == 0) return BURST_OK;
  if (hop->dtype == BURST_DTYPE_BF16) {
    // one kernel for every query range: lao_bwd4 walks whole 128-row dQ tiles of the
    // block and masks the rows of the first tile before q_begin (unaligned zigzag chunks)
    if (hop->head_dim == 128)
      return launch_bwd4_bf16<128>(hop, q, k, v, dout, stats, dq_acc, dk_acc, dv_acc, accumulate, st);
    return launch_bwd4_bf16<64>(hop, q, k, v, dout, stats, dq_acc, dk_acc, dv_acc, accumulate, st);
  }
  switch (hop->head_dim) {
    case 16: return launch_bwd_f32<16>(hop, q, k, v, dout, stats, dq_acc, dk_acc, dv_acc, accumulate, st);
    case 32: return launch_bwd_f32<32>(hop, q, k, v, dout, stats, dq_acc, dk_acc, dv_acc, accumulate, st);
    default: return launch_bwd_f32<64>(hop, q, k, v, dout, stats, dq_acc, dk_acc, dv_acc, accumulate, st);
  }
}

int burst_bwd_finalize(int dtype, int batch, int heads, int head_dim, int64_t n, const float* dq_acc,
                       const float* const* dk_parts, const float* const* dv_parts, int nparts, void* dq,
                       void* dk, void* dv, int32_t* flags, void* stream) {
  int rc = check_dims(dtype, batch, heads, head_dim, n);
  if (rc) return rc;
  if (nparts < 0 || nparts > 16) return fail(BURST_E_SHAPE, "nparts must be in [0, 16]");
  int* fl = flags_or_default(flags);
  if (n == 0) return BURST_OK;
  aux::Parts pk, pv;
  for (int i = 0; i < 16; ++i) {
    pk.p[i] = i < nparts ? dk_parts[i] : nullptr;
    pv.p[i] = i < nparts ? dv_parts[i] : nullptr;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (dq_acc) {
    aux::Parts pq{};
    pq.p[0] = dq_acc;
    launch_tl_rows(dtype, false, batch, heads, head_dim, n, pq, 1, dq, nullptr, nullptr, nullptr, fl, st);
  }
  if (nparts > 0) {
    launch_tl_rows(dtype, false, batch, heads, head_dim, n, pk, nparts, dk, nullptr, nullptr, nullptr, fl, st);
    launch_tl_rows(dtype, false, batch, heads, head_dim, n, pv, nparts, dv, nullptr, nullptr, nullptr, fl, st);
  }
  CHECK_LAUNCH();
  return BURST_OK;
}

int burst_tl_sum(int dtype, int batch, int heads, int head_dim, int64_t n, const float* const* parts,
                 int nparts, void* out, int32_t* flags, void* stream) {
  int rc = check_dims(dtype, batch, heads, head_dim, n);
  if (rc) return rc;
  if (nparts < 1 || nparts > 16) return fail(BURST_E_SHAPE, "nparts must be in [1, 16]");
  if (!out) return fail(BURST_E_SHAPE, "out must not be NULL");
  if (n == 0) return BURST_OK;
  aux::Parts pp;
  for (int i = 0; i < 16; ++i) pp.p[i] = i < nparts ? parts[i] : nullptr;
  launch_tl_rows(dtype, false, batch, heads, head_dim, n, pp, nparts, out, nullptr, nullptr, nullptr,
                 flags_or_default(flags), (cudaStream_t)stream);
  CHECK_LAUNCH();
  return BURST_OK;
}

int burst_tl_accumulate(int batch, int heads, int head_dim, int64_t n, float* acc, const float* part,
                        void* stream) {
  if (batch < 1 || heads < 1 || n < 0) return fail(BURST_E_SHAPE, "batch/heads must be positive, n >= 0");
  if (head_dim != 16 && head_dim != 32 && head_dim != 64 && head_dim != 128)
    return fail(BURST_E_UNSUPPORTED, "head_dim must be 16, 32, 64 or 128");
  if (!acc || !part) return fail(BURST_E_SHAPE, "acc and part must not be NULL");
  if ((reinterpret_cast<uintptr_t>(acc) | reinterpret_cast<uintptr_t>(part)) & 15)
    return fail(BURST_E_SHAPE, "TL workspaces must be 16-byte aligned");
  const int64_t n4 = (int64_t)burst_workspace_floats(batch, heads, head_dim, n) / 4;
  if (n4 == 0) return BURST_OK;
  aux::tl_accumulate_kernel<<<grid_for(n4, 256), 256, 0, (cudaStream_t)stream>>>(
      n4, reinterpret_cast<float4*>(acc), reinterpret_cast<const float4*>(part));
  CHECK_LAUNCH();
  return BURST_OK;
}

int burst_read_flags(void* stream, int* flags_out) {
  int* f = device_flags();
  if (!f) return fail(BURST_E_CUDA, "flag buffer allocation failed");
  int h = 0;
  CUDA_TRY(cudaMemcpyAsync(&h, f, sizeof(int), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  CUDA_TRY(cudaMemsetAsync(f, 0, sizeof(int), (cudaStream_t)stream));
  if (flags_out) *flags_out = h;
  return BURST_OK;
}

}  // extern "C"
