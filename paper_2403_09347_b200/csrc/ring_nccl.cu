// Ring transport: one NCCL communicator per ring, grouped send/recv per hop on
// the caller's (communication) stream.  Replaces the simulator's in-process
// RingChannel / DoubleBuffer hand-off (sim.py:281-332, lockstep rotation
// sim.py:560-568): device i sends to i+1 and receives from i-1 (sim.py:565).
//
// libnccl.so.2 is resolved at run time (dlopen) so the library loads on hosts
// without NCCL; PyTorch has normally loaded its bundled NCCL already and dlopen
// returns that instance.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/burst_b200.h"

namespace {

typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
constexpr int kNcclUint8 = 1;

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* candidates[] = {getenv("BURST_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    for (const char* c : candidates) {
      if (!c) continue;
      h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      a.why = "libnccl.so.2 not found (set BURST_NCCL_LIB)";
      return;
    }
#define SYM(field, name) a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name))
    SYM(GetUniqueId, "ncclGetUniqueId");
    SYM(CommInitRank, "ncclCommInitRank");
    SYM(CommDestroy, "ncclCommDestroy");
    SYM(Send, "ncclSend");
    SYM(Recv, "ncclRecv");
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.Send && a.Recv && a.GroupStart &&
           a.GroupEnd && a.GetErrorString;
    if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
  });
  return a;
}

struct Ring {
  ncclComm_t comm;
  int rank, world, device;
};

}  // namespace

// defined in capi.cu: records the message returned by burst_last_error()
int burst_internal_fail(int code, const std::string& msg);

static int ring_fail(int code, const std::string& m) { return burst_internal_fail(code, m); }

extern "C" {

int burst_ring_unique_id(void* out) {
  auto& a = api();
  if (!a.ok) return ring_fail(BURST_E_NCCL, a.why);
  ncclUniqueId id;
  ncclResult_t r = a.GetUniqueId(&id);
  if (r != 0) return ring_fail(BURST_E_NCCL, std::string("ncclGetUniqueId: ") + a.GetErrorString(r));
  memcpy(out, &id, sizeof(id));
  return BURST_OK;
}

int burst_ring_create(const void* uid, int rank, int world, int device, void** ring) {
  auto& a = api();
  if (!a.ok) return ring_fail(BURST_E_NCCL, a.why);
  if (world < 1 || rank < 0 || rank >= world || !ring) return ring_fail(BURST_E_SHAPE, "bad rank/world");
  if (cudaSetDevice(device) != cudaSuccess) return ring_fail(BURST_E_CUDA, "cudaSetDevice failed");
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  Ring* r = new Ring{nullptr, rank, world, device};
  ncclResult_t e = a.CommInitRank(&r->comm, world, id, rank);
  if (e != 0) {
    delete r;
    return ring_fail(BURST_E_NCCL, std::string("ncclCommInitRank: ") + a.GetErrorString(e));
  }
  *ring = r;
  return BURST_OK;
}

int burst_ring_exchange(void* ring, const void* send, void* recv, size_t bytes, int send_to,
                        int recv_from, void* stream) {
  auto& a = api();
  Ring* r = static_cast<Ring*>(ring);
  if (!r) return ring_fail(BURST_E_SHAPE, "null ring");
  if (send_to < 0 || send_to >= r->world || recv_from < 0 || recv_from >= r->world)
    return ring_fail(BURST_E_SHAPE, "peer out of range");
  cudaStream_t st = (cudaStream_t)stream;
  ncclResult_t e = a.GroupStart();
  if (e == 0 && send) e = a.Send(send, bytes, kNcclUint8, send_to, r->comm, st);
  if (e == 0 && recv) e = a.Recv(recv, bytes, kNcclUint8, recv_from, r->comm, st);
  ncclResult_t e2 = a.GroupEnd();
  if (e != 0 || e2 != 0)
    return ring_fail(BURST_E_NCCL, std::string("ring exchange: ") + a.GetErrorString(e ? e : e2));
  return BURST_OK;
}

int burst_ring_sendrecv(void* ring, const burst_p2p* ops, int nops, void* stream) {
  auto& a = api();
  Ring* r = static_cast<Ring*>(ring);
  if (!r) return ring_fail(BURST_E_SHAPE, "null ring");
  if (nops < 0 || (nops > 0 && !ops)) return ring_fail(BURST_E_SHAPE, "bad op list");
  for (int i = 0; i < nops; ++i)
    if (ops[i].peer < 0 || ops[i].peer >= r->world) return ring_fail(BURST_E_SHAPE, "peer out of range");
  cudaStream_t st = (cudaStream_t)stream;
  ncclResult_t e = a.GroupStart();
  for (int i = 0; e == 0 && i < nops; ++i) {
    if (ops[i].bytes == 0) continue;
    if (ops[i].is_send)
      e = a.Send(ops[i].buf, ops[i].bytes, kNcclUint8, ops[i].peer, r->comm, st);
    else
      e = a.Recv(ops[i].buf, ops[i].bytes, kNcclUint8, ops[i].peer, r->comm, st);
  }
  ncclResult_t e2 = a.GroupEnd();
  if (e != 0 || e2 != 0)
    return ring_fail(BURST_E_NCCL, std::string("ring sendrecv: ") + a.GetErrorString(e ? e : e2));
  return BURST_OK;
}

int burst_ring_destroy(void* ring) {
  auto& a = api();
  Ring* r = static_cast<Ring*>(ring);
  if (!r) return BURST_OK;
  if (a.ok && r->comm) a.CommDestroy(r->comm);
  delete r;
  return BURST_OK;
}

}  // extern "C"
