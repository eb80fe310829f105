// Ring transport: one NCCL communicator per ring, grouped send/recv per hop on
// the caller's (communication) stream.  Replaces the simulator's in-process
// RingChannel / DoubleBuffer hand-off (sim.py:281-332, lockstep rotation
// sim.py:560-568): device i sends to i+1 and receives from i-1 (sim.py:565).
//
// Failure detection (the reference's DeadlockError on a stalled channel,
// sim.py:290-310, and on a run that stops making progress, sim.py:622-631):
// the communicator is created NON-BLOCKING; every exchange records a CUDA event on
// the comm stream after its grouped send/recv, and a watchdog thread per ring
// polls those events and ncclCommGetAsyncError.  If no posted exchange completes
// within `timeout_s` of the last observed progress, or NCCL reports an
// asynchronous error, the watchdog calls ncclCommAbort -- which makes the stuck
// NCCL kernels return, so a caller blocked in a stream synchronise wakes up --
// and every later call on the ring returns BURST_E_DEADLOCK / BURST_E_NCCL.
// Joining (ncclCommInitRankConfig) is bounded by the same timeout.
//
// libnccl.so.2 is resolved at run time (dlopen) so the library loads on hosts
// without NCCL; PyTorch has normally loaded its bundled NCCL already and dlopen
// returns that instance.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <thread>

#include "../../include/burst_b200.h"

namespace {

typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
constexpr int kNcclUint8 = 1;
constexpr ncclResult_t kNcclSuccess = 0, kNcclInProgress = 7;
constexpr int kUndefInt = (int)0x80000000;

// ncclConfig_t as of NCCL 2.28 (nccl.h ncclConfig_v22800).  `version` is set to the
// loaded library's version so an older NCCL reads only the fields it knows.
struct NcclConfig {
  size_t size;
  unsigned int magic;
  unsigned int version;
  int blocking, cgaClusterSize, minCTAs, maxCTAs;
  const char* netName;
  int splitShare, trafficClass;
  const char* commName;
  int collnetEnable, CTAPolicy, shrinkShare, nvlsCTAs, nChannelsPerNetPeer, nvlinkCentricSched;
};

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  ncclResult_t (*CommInitRankConfig)(ncclComm_t*, int, ncclUniqueId, int, NcclConfig*) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
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
    SYM(GetVersion, "ncclGetVersion");
    SYM(CommInitRankConfig, "ncclCommInitRankConfig");
    SYM(CommGetAsyncError, "ncclCommGetAsyncError");
    SYM(CommAbort, "ncclCommAbort");
    SYM(CommDestroy, "ncclCommDestroy");
    SYM(Send, "ncclSend");
    SYM(Recv, "ncclRecv");
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    a.ok = a.GetUniqueId && a.GetVersion && a.CommInitRankConfig && a.CommGetAsyncError &&
           a.CommAbort && a.CommDestroy && a.Send && a.Recv && a.GroupStart && a.GroupEnd &&
           a.GetErrorString;
    if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol (NCCL >= 2.14 needed)";
  });
  return a;
}

using Clock = std::chrono::steady_clock;

struct Ring {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1, device = 0;
  double timeout_s = 600.0;
  std::mutex mu;
  std::deque<cudaEvent_t> pending;        // one event per posted exchange, in order
  std::deque<cudaEvent_t> free_events;
  uint64_t posted = 0, completed = 0;
  Clock::time_point last_progress = Clock::now();
  std::atomic<int> failed{0};             // BURST_E_DEADLOCK / BURST_E_NCCL once aborted
  std::string why;
  std::atomic<bool> stop{false};
  std::thread watchdog;
};

// Retire completed exchanges; abort on a stall or an asynchronous NCCL error.
// Called with r->mu held.  Returns the failure code (0 = healthy).
int poll_locked(Ring* r) {
  if (r->failed.load()) return r->failed.load();
  while (!r->pending.empty()) {
    cudaError_t q = cudaEventQuery(r->pending.front());
    if (q == cudaErrorNotReady) break;
    r->free_events.push_back(r->pending.front());
    r->pending.pop_front();
    ++r->completed;
    r->last_progress = Clock::now();
    if (q != cudaSuccess) {
      r->why = std::string("ring exchange failed on the device: ") + cudaGetErrorString(q);
      r->failed = BURST_E_CUDA;
      return r->failed;
    }
  }
  auto& a = api();
  ncclResult_t st = kNcclSuccess;
  if (!r->comm) return 0;
  if (a.CommGetAsyncError(r->comm, &st) == kNcclSuccess && st != kNcclSuccess && st != kNcclInProgress) {
    r->why = std::string("NCCL asynchronous error: ") + a.GetErrorString(st);
    a.CommAbort(r->comm);
    r->comm = nullptr;
    r->failed = BURST_E_NCCL;
    return r->failed;
  }
  if (!r->pending.empty()) {
    const double idle = std::chrono::duration<double>(Clock::now() - r->last_progress).count();
    if (idle > r->timeout_s) {
      r->why = "DeadlockError: ring rank " + std::to_string(r->rank) + " of " +
               std::to_string(r->world) + ": exchange #" + std::to_string(r->completed) +
               " made no progress within " + std::to_string(r->timeout_s) +
               " s (peer stalled or gone); communicator aborted";
      a.CommAbort(r->comm);
      r->comm = nullptr;
      r->failed = BURST_E_DEADLOCK;
      return r->failed;
    }
  } else {
    r->last_progress = Clock::now();
  }
  return 0;
}

void watchdog_main(Ring* r) {
  cudaSetDevice(r->device);
  while (!r->stop.load()) {
    {
      std::lock_guard<std::mutex> lk(r->mu);
      if (poll_locked(r)) return;
    }
    std::this_thread::sleep_for(std::chrono::milliseconds(2));
  }
}

}  // namespace

// defined in capi.cu: records the message returned by burst_last_error()
int burst_internal_fail(int code, const std::string& msg);

static int ring_fail(int code, const std::string& m) { return burst_internal_fail(code, m); }

static int ring_failed(Ring* r) {
  const int f = r->failed.load();
  return f ? ring_fail(f, r->why) : BURST_OK;
}

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

int burst_ring_create(const void* uid, int rank, int world, int device, double timeout_s,
                      void** ring) {
  auto& a = api();
  if (!a.ok) return ring_fail(BURST_E_NCCL, a.why);
  if (world < 1 || rank < 0 || rank >= world || !ring || !uid) return ring_fail(BURST_E_SHAPE, "bad rank/world");
  if (!(timeout_s > 0)) return ring_fail(BURST_E_SHAPE, "timeout_s must be positive");
  if (cudaSetDevice(device) != cudaSuccess) return ring_fail(BURST_E_CUDA, "cudaSetDevice failed");
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  int version = 0;
  a.GetVersion(&version);
  NcclConfig cfg{sizeof(NcclConfig), 0xcafebeefu, (unsigned)version, 0 /* non-blocking */,
                 kUndefInt, kUndefInt, kUndefInt, nullptr, kUndefInt, kUndefInt, nullptr,
                 kUndefInt, kUndefInt, kUndefInt, kUndefInt, kUndefInt, kUndefInt};
  Ring* r = new Ring;
  r->rank = rank; r->world = world; r->device = device; r->timeout_s = timeout_s;
  ncclResult_t e = a.CommInitRankConfig(&r->comm, world, id, rank, &cfg);
  const auto t0 = Clock::now();
  ncclResult_t st = e;
  while (e == kNcclSuccess || e == kNcclInProgress) {
    if (a.CommGetAsyncError(r->comm, &st) != kNcclSuccess) break;
    if (st != kNcclInProgress) break;
    if (std::chrono::duration<double>(Clock::now() - t0).count() > timeout_s) {
      a.CommAbort(r->comm);
      delete r;
      return ring_fail(BURST_E_DEADLOCK, "DeadlockError: ring rank " + std::to_string(rank) + " of " +
                                             std::to_string(world) + ": peers did not join within " +
                                             std::to_string(timeout_s) + " s; communicator aborted");
    }
    std::this_thread::sleep_for(std::chrono::milliseconds(1));
  }
  if ((e != kNcclSuccess && e != kNcclInProgress) || st != kNcclSuccess) {
    const ncclResult_t bad = (e != kNcclSuccess && e != kNcclInProgress) ? e : st;
    if (r->comm) a.CommAbort(r->comm);
    delete r;
    return ring_fail(BURST_E_NCCL, std::string("ncclCommInitRankConfig: ") + a.GetErrorString(bad));
  }
  r->watchdog = std::thread(watchdog_main, r);
  *ring = r;
  return BURST_OK;
}

// Wait for the non-blocking group launch to be enqueued.
static int finish_group(Ring* r, ncclResult_t e, const char* what) {
  auto& a = api();
  if (e == kNcclInProgress) {
    ncclResult_t st = kNcclInProgress;
    while (a.CommGetAsyncError(r->comm, &st) == kNcclSuccess && st == kNcclInProgress) std::this_thread::yield();
    e = st;
  }
  if (e != kNcclSuccess) return ring_fail(BURST_E_NCCL, std::string(what) + ": " + a.GetErrorString(e));
  return BURST_OK;
}

static int record_exchange(Ring* r, cudaStream_t st) {
  cudaEvent_t ev;
  if (!r->free_events.empty()) {
    ev = r->free_events.front();
    r->free_events.pop_front();
  } else if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
    return ring_fail(BURST_E_CUDA, "cudaEventCreate failed");
  }
  if (cudaEventRecord(ev, st) != cudaSuccess) return ring_fail(BURST_E_CUDA, "cudaEventRecord failed");
  if (r->pending.empty()) r->last_progress = Clock::now();
  r->pending.push_back(ev);
  ++r->posted;
  return BURST_OK;
}

int burst_ring_sendrecv(void* ring, const burst_p2p* ops, int nops, void* stream) {
  auto& a = api();
  Ring* r = static_cast<Ring*>(ring);
  if (!r) return ring_fail(BURST_E_SHAPE, "null ring");
  if (nops < 0 || (nops > 0 && !ops)) return ring_fail(BURST_E_SHAPE, "bad op list");
  for (int i = 0; i < nops; ++i)
    if (ops[i].peer < 0 || ops[i].peer >= r->world) return ring_fail(BURST_E_SHAPE, "peer out of range");
  std::lock_guard<std::mutex> lk(r->mu);
  if (int rc = ring_failed(r)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  ncclResult_t e = a.GroupStart();
  for (int i = 0; e == kNcclSuccess && i < nops; ++i) {
    if (ops[i].bytes == 0) continue;
    if (ops[i].is_send)
      e = a.Send(ops[i].buf, ops[i].bytes, kNcclUint8, ops[i].peer, r->comm, st);
    else
      e = a.Recv(ops[i].buf, ops[i].bytes, kNcclUint8, ops[i].peer, r->comm, st);
  }
  ncclResult_t e2 = a.GroupEnd();
  if (e != kNcclSuccess) return ring_fail(BURST_E_NCCL, std::string("ring sendrecv: ") + a.GetErrorString(e));
  if (int rc = finish_group(r, e2, "ring sendrecv")) return rc;
  return record_exchange(r, st);
}

int burst_ring_exchange(void* ring, const void* send, void* recv, size_t bytes, int send_to,
                        int recv_from, void* stream) {
  Ring* r = static_cast<Ring*>(ring);
  if (!r) return ring_fail(BURST_E_SHAPE, "null ring");
  burst_p2p ops[2];
  int n = 0;
  if (send) ops[n++] = burst_p2p{const_cast<void*>(send), bytes, send_to, 1};
  if (recv) ops[n++] = burst_p2p{recv, bytes, recv_from, 0};
  return burst_ring_sendrecv(ring, ops, n, stream);
}

int burst_ring_poll(void* ring, uint64_t* posted, uint64_t* completed) {
  Ring* r = static_cast<Ring*>(ring);
  if (!r) return ring_fail(BURST_E_SHAPE, "null ring");
  std::lock_guard<std::mutex> lk(r->mu);
  poll_locked(r);
  if (posted) *posted = r->posted;
  if (completed) *completed = r->completed;
  return ring_failed(r);
}

int burst_ring_wait(void* ring) {
  Ring* r = static_cast<Ring*>(ring);
  if (!r) return ring_fail(BURST_E_SHAPE, "null ring");
  for (;;) {
    {
      std::lock_guard<std::mutex> lk(r->mu);
      poll_locked(r);
      if (int rc = ring_failed(r)) return rc;
      if (r->pending.empty()) return BURST_OK;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
}

int burst_ring_destroy(void* ring) {
  auto& a = api();
  Ring* r = static_cast<Ring*>(ring);
  if (!r) return BURST_OK;
  r->stop = true;
  if (r->watchdog.joinable()) r->watchdog.join();
  cudaSetDevice(r->device);
  if (a.ok && r->comm) {    // an aborted communicator is already released (comm == NULL)
    for (cudaEvent_t ev : r->pending) cudaEventSynchronize(ev);
    a.CommDestroy(r->comm);
  }
  for (cudaEvent_t ev : r->pending) cudaEventDestroy(ev);
  for (cudaEvent_t ev : r->free_events) cudaEventDestroy(ev);
  delete r;
  return BURST_OK;
}

}  // extern "C"
