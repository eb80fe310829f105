// Zero-SM ring transport: copy-engine peer copies into CUDA IPC
// mailboxes, ordered by device-side sequence flags.  NCCL send/recv kernels occupy
// SMs that a full-grid attention kernel also wants; cudaMemcpyAsync between
// device buffers (over NVLink for peers on other GPUs) runs on the copy engines
// and uses no SM, and the flag handshake (cuStreamWriteValue32 into a local
// staging word + a 4-byte copy into the peer's flag array; cuStreamWaitValue32 on
// our own flags) runs in the stream front end, so an exchange needs no host
// round trip at all.  The protocol (mailbox layout, flags, sequence numbers)
// lives in ring.IpcTransport; this file wraps the CUDA calls it needs behind the
// C ABI.
//
// Replaces the same simulator pieces as ring_nccl.cu: RingChannel send/recv and
// DoubleBuffer (sim.py:281-332).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/burst_b200.h"

int burst_internal_fail(int code, const std::string& msg);   // capi.cu

namespace {
int cuda_fail(const char* what, cudaError_t e) {
  return burst_internal_fail(BURST_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Stream memory operations (driver API) through the runtime's entry-point query, so
// the library does not link libcuda directly.
using WriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WriteFn g_write = nullptr;
WaitFn g_wait = nullptr;

bool load_memops() {
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_write = reinterpret_cast<WriteFn>(p);
    p = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_wait = reinterpret_cast<WaitFn>(p);
  });
  return g_write && g_wait;
}

int cu_fail(const char* what, CUresult r) {
  return burst_internal_fail(BURST_E_CUDA, std::string(what) + " failed (CUresult " +
                                               std::to_string((int)r) + ")");
}
}  // namespace

extern "C" {

size_t burst_ipc_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

// Mailboxes get their own cudaMalloc allocation: an IPC handle names a whole
// allocation, so a sub-allocation of a caching allocator would open at the wrong base.
// The memory is zeroed (sequence flags start at 0).
int burst_ipc_alloc(size_t bytes, void** dev_ptr) {
  if (!dev_ptr) return burst_internal_fail(BURST_E_SHAPE, "null pointer");
  cudaError_t e = cudaMalloc(dev_ptr, bytes ? bytes : 1);
  if (e != cudaSuccess) return cuda_fail("cudaMalloc", e);
  e = cudaMemset(*dev_ptr, 0, bytes ? bytes : 1);
  return e == cudaSuccess ? BURST_OK : cuda_fail("cudaMemset", e);
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

// Publish `value` into a 4-byte flag that may live in a peer's memory (IPC-mapped,
// NVLink for another GPU): cuStreamWriteValue32 into the local staging word
// `stage`, then a copy-engine copy stage -> flag.  Both are ordered after every
// earlier operation of `stream` (the data pushes the flag announces).
int burst_signal_u32(void* stream, void* flag, void* stage, uint32_t value) {
  if (!flag || !stage) return burst_internal_fail(BURST_E_SHAPE, "null flag pointer");
  if (!load_memops()) return burst_internal_fail(BURST_E_CUDA, "stream memory operations unavailable");
  // a flag on the stream's own device (a peer process on the same GPU, or our own
  // memory) takes the write directly; a flag in another GPU's memory goes through
  // the staging word and a copy-engine copy over NVLink
  int cur = -1;
  cudaPointerAttributes pa;
  const bool local = cudaGetDevice(&cur) == cudaSuccess &&
                     cudaPointerGetAttributes(&pa, flag) == cudaSuccess &&
                     pa.type == cudaMemoryTypeDevice && pa.device == cur;
  CUresult r = g_write((CUstream)stream, (CUdeviceptr)(local ? flag : stage), value, 0);
  if (r != CUDA_SUCCESS) return cu_fail("cuStreamWriteValue32", r);
  if (local || flag == stage) return BURST_OK;
  cudaError_t e = cudaMemcpyAsync(flag, stage, 4, cudaMemcpyDeviceToDevice, (cudaStream_t)stream);
  return e == cudaSuccess ? BURST_OK : cuda_fail("cudaMemcpyAsync", e);
}

// Block `stream` (in the stream front end: no SM, no host thread) until the 4-byte
// flag in OUR memory reaches `value` ((int32)(flag - value) >= 0, wrap-safe).
int burst_wait_u32(void* stream, void* flag, uint32_t value) {
  if (!flag) return burst_internal_fail(BURST_E_SHAPE, "null flag pointer");
  if (!load_memops()) return burst_internal_fail(BURST_E_CUDA, "stream memory operations unavailable");
  CUresult r = g_wait((CUstream)stream, (CUdeviceptr)flag, value, CU_STREAM_WAIT_VALUE_GEQ);
  return r == CUDA_SUCCESS ? BURST_OK : cu_fail("cuStreamWaitValue32", r);
}

}  // extern "C"

// ------------------------------------------------------------------ IPC ring
// One exchange of ring.IpcTransport posted by a single call (no host round trip,
// a few microseconds of host time): the protocol of the class docstring, executed
// here so Python issues one C call per exchange.
namespace {
struct IpcRing {
  int rank = 0, world = 0;
  uint8_t* flags = nullptr;            // mine: [world][2 slots][ready, free] uint32
  uint8_t* stage = nullptr;            // local staging words, same shape
  std::vector<uint8_t*> peer_flags, peer_mail;
  uint8_t* mail = nullptr;             // mine: 2 slots
  size_t slot_bytes = 0;
  size_t caps[3] = {0, 0, 0};
  uint32_t e = 0;                      // exchanges posted
};
inline uint8_t* flag_at(uint8_t* base, int peer, int slot, int kind) {
  return base + ((size_t)(peer * 2 + slot) * 2 + kind) * 4;
}
size_t tag_off(const IpcRing* r, int tag) {
  size_t o = 0;
  for (int t = 0; t < tag; ++t) o += r->caps[t];
  return o;
}
}  // namespace

extern "C" {

int burst_ipc_ring_create(int rank, int world, void* flags, void* stage, void** out) {
  if (!out || !flags || !stage || world < 1 || rank < 0 || rank >= world)
    return burst_internal_fail(BURST_E_SHAPE, "bad IPC ring arguments");
  auto* r = new IpcRing();
  r->rank = rank;
  r->world = world;
  r->flags = static_cast<uint8_t*>(flags);
  r->stage = static_cast<uint8_t*>(stage);
  r->peer_flags.assign(world, nullptr);
  r->peer_mail.assign(world, nullptr);
  *out = r;
  return BURST_OK;
}

int burst_ipc_ring_set_peer(void* ring, int peer, void* peer_flags, void* peer_mail) {
  auto* r = static_cast<IpcRing*>(ring);
  if (!r || peer < 0 || peer >= r->world) return burst_internal_fail(BURST_E_SHAPE, "bad peer");
  if (peer_flags) r->peer_flags[peer] = static_cast<uint8_t*>(peer_flags);
  r->peer_mail[peer] = static_cast<uint8_t*>(peer_mail);
  return BURST_OK;
}

int burst_ipc_ring_set_mailbox(void* ring, void* mail, size_t slot_bytes, const uint64_t* caps) {
  auto* r = static_cast<IpcRing*>(ring);
  if (!r || !caps) return burst_internal_fail(BURST_E_SHAPE, "bad mailbox arguments");
  r->mail = static_cast<uint8_t*>(mail);
  r->slot_bytes = slot_bytes;
  for (int t = 0; t < 3; ++t) r->caps[t] = (size_t)caps[t];
  return BURST_OK;
}

int burst_ipc_ring_exchange(void* ring, const burst_ipc_op* ops, int nops, void* stream) {
  auto* r = static_cast<IpcRing*>(ring);
  if (!r || (nops > 0 && !ops)) return burst_internal_fail(BURST_E_SHAPE, "bad exchange arguments");
  if (!r->mail) return burst_internal_fail(BURST_E_DESYNC, "IPC exchange before the mailbox is reserved");
  const int s = (int)(r->e & 1u);
  const uint32_t q = r->e + 1u;
  ++r->e;
  std::vector<int> from, to;
  for (int i = 0; i < nops; ++i) {
    const auto& o = ops[i];
    if (o.peer < 0 || o.peer >= r->world || o.peer == r->rank || o.tag < 0 || o.tag > 2)
      return burst_internal_fail(BURST_E_SHAPE, "bad IPC op (peer or tag)");
    auto& v = o.is_send ? to : from;
    if (std::find(v.begin(), v.end(), o.peer) == v.end()) v.push_back(o.peer);
  }
  // 1. our slot s is free for every sender of this exchange
  for (int p : from) {
    int rc = burst_signal_u32(stream, flag_at(r->peer_flags[p], r->rank, s, 1),
                              flag_at(r->stage, p, s, 1), q);
    if (rc) return rc;
  }
  // 2. pushes into the receivers' slots (copy engines), then their ready flags
  for (int d : to) {
    int rc = burst_wait_u32(stream, flag_at(r->flags, d, s, 1), q);
    if (rc) return rc;
    size_t offs[3] = {0, 0, 0};
    uint8_t* base = r->peer_mail[d] + (size_t)s * r->slot_bytes;
    for (int i = 0; i < nops; ++i) {
      const auto& o = ops[i];
      if (!o.is_send || o.peer != d) continue;
      if (offs[o.tag] + o.bytes > r->caps[o.tag])
        return burst_internal_fail(BURST_E_DESYNC, "IPC payload exceeds the receiver's reserved region");
      rc = burst_copy_async(base + tag_off(r, o.tag) + offs[o.tag], o.buf, o.bytes, stream);
      if (rc) return rc;
      offs[o.tag] += o.bytes;
    }
    rc = burst_signal_u32(stream, flag_at(r->peer_flags[d], r->rank, s, 0), flag_at(r->stage, d, s, 0), q);
    if (rc) return rc;
  }
  // 3. wait for our senders; receives not already in place are copied out
  for (int p : from) {
    int rc = burst_wait_u32(stream, flag_at(r->flags, p, s, 0), q);
    if (rc) return rc;
  }
  size_t offs[3] = {0, 0, 0};
  uint8_t* base = r->mail + (size_t)s * r->slot_bytes;
  for (int i = 0; i < nops; ++i) {
    const auto& o = ops[i];
    if (o.is_send) continue;
    uint8_t* src = base + tag_off(r, o.tag) + offs[o.tag];
    if (offs[o.tag] + o.bytes > r->caps[o.tag])
      return burst_internal_fail(BURST_E_DESYNC, "IPC receive exceeds the reserved region");
    offs[o.tag] += o.bytes;
    if (o.buf != src) {
      int rc = burst_copy_async(o.buf, src, o.bytes, stream);
      if (rc) return rc;
    }
  }
  return BURST_OK;
}

int burst_ipc_ring_destroy(void* ring) {
  delete static_cast<IpcRing*>(ring);
  return BURST_OK;
}

}  // extern "C"
