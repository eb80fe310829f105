// Zero-SM ring transport: copy-engine peer copies into CUDA IPC
// mailboxes, ordered by interprocess CUDA events.  NCCL send/recv kernels occupy
// SMs that a full-grid attention kernel also wants; cudaMemcpyAsync between
// device buffers (over NVLink for peers on other GPUs) runs on the copy engines
// and uses no SM.  The host protocol (mailbox sizing, handle exchange, the
// per-exchange barrier) lives in ring.IpcTransport; this file only wraps the
// CUDA runtime calls it needs behind the C ABI.
//
// Replaces the same simulator pieces as ring_nccl.cu: RingChannel send/recv and
// DoubleBuffer (sim.py:281-332).
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "../../include/burst_b200.h"

int burst_internal_fail(int code, const std::string& msg);   // capi.cu

namespace {
int cuda_fail(const char* what, cudaError_t e) {
  return burst_internal_fail(BURST_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace

extern "C" {

size_t burst_ipc_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

// Mailboxes get their own cudaMalloc allocation: an IPC handle names a whole
// allocation, so a sub-allocation of a caching allocator would open at the wrong base.
int burst_ipc_alloc(size_t bytes, void** dev_ptr) {
  if (!dev_ptr) return burst_internal_fail(BURST_E_SHAPE, "null pointer");
  cudaError_t e = cudaMalloc(dev_ptr, bytes ? bytes : 1);
  return e == cudaSuccess ? BURST_OK : cuda_fail("cudaMalloc", e);
}

int burst_ipc_free(void* dev_ptr) {
  cudaError_t e = cudaFree(dev_ptr);
  return e == cudaSuccess ? BURST_OK : cuda_fail("cudaFree", e);
}

int burst_ipc_mem_handle(void* dev_ptr, void* out_handle) {
  if (!dev_ptr || !out_handle) return burst_internal_fail(BURST_E_SHAPE, "null pointer");
  cudaError_t e = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(out_handle), dev_ptr);
  return e == cudaSuccess ? BURST_OK : cuda_fail("cudaIpcGetMemHandle", e);
}

int burst_ipc_open_mem(const void* handle, void** dev_ptr) {
  if (!handle || !dev_ptr) return burst_internal_fail(BURST_E_SHAPE, "null pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? BURST_OK : cuda_fail("cudaIpcOpenMemHandle", e);
}

int burst_ipc_close_mem(void* dev_ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  return e == cudaSuccess ? BURST_OK : cuda_fail("cudaIpcCloseMemHandle", e);
}

int burst_ipc_event_create(void** event, void* out_handle) {
  if (!event || !out_handle) return burst_internal_fail(BURST_E_SHAPE, "null pointer");
  cudaEvent_t ev;
  cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming | cudaEventInterprocess);
  if (e != cudaSuccess) return cuda_fail("cudaEventCreateWithFlags", e);
  e = cudaIpcGetEventHandle(reinterpret_cast<cudaIpcEventHandle_t*>(out_handle), ev);
  if (e != cudaSuccess) return cuda_fail("cudaIpcGetEventHandle", e);
  *event = ev;
  return BURST_OK;
}

int burst_ipc_event_open(const void* handle, void** event) {
  if (!handle || !event) return burst_internal_fail(BURST_E_SHAPE, "null pointer");
  cudaIpcEventHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaEvent_t ev;
  cudaError_t e = cudaIpcOpenEventHandle(&ev, h);
  if (e != cudaSuccess) return cuda_fail("cudaIpcOpenEventHandle", e);
  *event = ev;
  return BURST_OK;
}

int burst_event_record(void* event, void* stream) {
  cudaError_t e = cudaEventRecord((cudaEvent_t)event, (cudaStream_t)stream);
  return e == cudaSuccess ? BURST_OK : cuda_fail("cudaEventRecord", e);
}

int burst_stream_wait_event(void* stream, void* event) {
  cudaError_t e = cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)event, 0);
  return e == cudaSuccess ? BURST_OK : cuda_fail("cudaStreamWaitEvent", e);
}

int burst_event_destroy(void* event) {
  cudaError_t e = cudaEventDestroy((cudaEvent_t)event);
  return e == cudaSuccess ? BURST_OK : cuda_fail("cudaEventDestroy", e);
}

// Device-to-device copy on `stream` by the copy engines (peer memory included).
int burst_copy_async(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes == 0) return BURST_OK;
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream);
  return e == cudaSuccess ? BURST_OK : cuda_fail("cudaMemcpyAsync", e);
}

}  // extern "C"
