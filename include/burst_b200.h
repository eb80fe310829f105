/* burst_b200.h -- C ABI of the B200-native BurstAttention hot path.
 *
 * Every entry point is asynchronous on the caller's CUDA stream (passed as an
 * opaque `void*` cudaStream_t), takes plain device pointers and sizes, never
 * allocates, and returns 0 or a BURST_E_* code (message via burst_last_error).
 * The error codes mirror the reference taxonomy (pkg/src/burstsim/errors.py:4-33).
 *
 * Reference interfaces replaced (all /root/reference/pkg/src/burstsim/):
 *   burst_lao_fwd        local_attn.local_forward_tiled   (local_attn.py:207-248)
 *                        + PartialAttn.merge               (local_attn.py:101-120)
 *                        = ring.forward_step hop merge     (ring.py:158-181)
 *   burst_fwd_finalize   PartialAttn.finalize / ring.finalize_forward
 *                                                          (local_attn.py:127-135, ring.py:184-188)
 *   burst_bwd_preprocess ring.init_backward D = rowsum(dO*O) (ring.py:195-218)
 *   burst_lao_bwd        local_attn.local_backward         (local_attn.py:255-289)
 *                        = ring.backward_step accumulation (ring.py:221-242)
 *   burst_bwd_finalize   sim._collect gradient assembly    (sim.py:450-471)
 *   burst_tl_sum         same, for travelling-query dQ contributions (ring.py:65-83)
 *   burst_tl_accumulate  in-place accumulation of a received contribution (ring.py:239-241)
 *   burst_ring_*         sim.RingChannel send/recv, DoubleBuffer (sim.py:281-332)
 *   burst_ipc_*, burst_copy_async, burst_event_* / burst_stream_wait_event
 *                        the same hand-off over copy engines (zero SM), SURVEY f1
 *
 * Tensor layouts (row-major, contiguous):
 *   q, k, v, o, dout, dq, dk, dv : [batch, n, heads, head_dim]  (bf16 or f32)
 *   lse, m, l                    : [batch, heads, n] f32 (lse natural log, m log2 units)
 *   o_acc, dq_acc, dk/dv partials: f32 "TL" workspace, burst_workspace_floats()
 *                                  elements, layout [B*H][ceil(n/128)][D/4][128][4]
 */
#ifndef BURST_B200_H
#define BURST_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define BURST_API __attribute__((visibility("default")))
#else
#define BURST_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum {
  BURST_OK = 0,
  BURST_E_SHAPE = 1,      /* ShapeError */
  BURST_E_MASK = 2,       /* MaskError: a query row saw no key */
  BURST_E_NONFINITE = 3,  /* NonFiniteError */
  BURST_E_ORDER = 4,      /* MissingForwardError */
  BURST_E_CUDA = 5,
  BURST_E_NCCL = 6,
  BURST_E_DEADLOCK = 7,   /* DeadlockError */
  BURST_E_UNSUPPORTED = 8,
  BURST_E_DESYNC = 9      /* RingDesyncError: an exchange that does not fit the ring's layout */
};

enum { BURST_DTYPE_BF16 = 0, BURST_DTYPE_F32 = 1 };

/* Global position of local row i: i < seg_len ? pos0 + i : pos1 + (i - seg_len).
 * Monotone (pos0 + seg_len <= pos1).  Contiguous shards use one segment
 * (seg_len >= n); zigzag shards hold chunks r and 2G-1-r. */
typedef struct {
  int64_t pos0, pos1, seg_len;
} burst_posmap;

/* One hop: the pinned query block (n_q rows) against a visiting key/value block
 * (n_k rows).  Only query rows [q_begin, q_begin+q_len) and key rows
 * [k_begin, k_begin+k_len) participate (zigzag hop classes).  With `causal`,
 * key j is visible to query i iff k_map(j) <= q_map(i) (masking.py:116-117).
 * With `grid_skip` != NULL (BlockGrid, masking.py:33-63 and 120-128), key j is
 * also hidden from query i when cell (q_map(i) / grid_qcell, k_map(j) / grid_kcell)
 * is skipped: grid_skip is a device array of grid_nqb * grid_nkb bytes, row-major
 * over (query cell, key cell), 1 = skipped. */
typedef struct {
  int32_t batch, heads, head_dim, dtype;
  int64_t n_q, n_k;
  int64_t q_begin, q_len, k_begin, k_len;
  float softmax_scale;
  int32_t causal;
  burst_posmap q_map, k_map;
  const uint8_t* grid_skip;
  int32_t grid_nqb, grid_nkb;
  int64_t grid_qcell, grid_kcell;
  /* Device int32 error word of the pass this hop belongs to (NULL = the per-device
   * default word of burst_read_flags).  Kernels OR in bit 0 (a row with no visible
   * key -> MaskError), bit 1 (non-finite output -> NonFiniteError), bit 2 (launch
   * could not run -> CudaError). */
  int32_t* flags;
  /* Deterministic gradients (optional): non-NULL selects the bit-reproducible bf16
   * backward (the reference's bitwise executor equivalence, pkg/tests/test_sim.py:
   * 280-295): burst_lao_bwd then computes dK/dV in the key-stationary kernel and dQ in
   * a query-stationary kernel that accumulates each dQ row over the key tiles in order
   * and adds it to dq_acc once -- no order-dependent fp32 reduction is left.  The
   * device int32 array (batch * heads * ceil(n_q/128) words) is reserved scratch.
   * NULL = fastest (unordered fp32 dQ reductions).  The f32 path is always ordered. */
  int32_t* dq_order;
  /* Key-tile visiting order of the bf16 forward (optional; local_forward_tiled's
   * key_tile_order, local_attn.py:212-225): device int32 permutation of the hop's
   * ceil(k_len/128) key tiles (128 keys each, counted from k_begin), read by every CTA
   * (not validated on the device).  The online-softmax merge is order-independent up
   * to rounding.  NULL = ascending.  The f32 path ignores it. */
  const int32_t* key_order;
} burst_hop;

/* Elements (float) of one TL workspace for [batch, n, heads, head_dim]. */
BURST_API size_t burst_workspace_floats(int batch, int heads, int head_dim, int64_t n);

/* LAO forward of one hop fused with the GAO merge into the running state
 * (o_acc TL, m/l in log2 units).  first_hop: ignore the incoming state.
 * finalize: normalise and write o_out (dtype) and lse_out instead of the state. */
BURST_API int burst_lao_fwd(const burst_hop* hop, const void* q, const void* k, const void* v, float* o_acc,
                  float* m, float* l, void* o_out, float* lse_out, int first_hop, int finalize,
                  void* stream);

/* Normalise a running state: o_out = o_acc / l, lse = ln-domain(m, l).  `flags`:
 * error word (see burst_hop.flags; NULL = per-device default). */
BURST_API int burst_fwd_finalize(int dtype, int batch, int heads, int head_dim, int64_t n,
                       const float* o_acc, const float* m, const float* l, void* o_out,
                       float* lse_out, int32_t* flags, void* stream);

/* Backward stats for every (b, h, row) of a [batch, n] query block, packed as
 * stats[0][B*H][ceil(n/128)*128] = lse * log2(e) and stats[1][...] = D =
 * rowsum(dout * o) (padded rows: +inf / 0); also zeroes dq_acc (TL) if given.
 * `stats` holds 2 * batch * heads * ceil(n/128) * 128 floats (burst_lao_bwd reads
 * whole 128-row tiles of the block, never past the last tile). */
BURST_API int burst_bwd_preprocess(int dtype, int batch, int heads, int head_dim, int64_t n, const void* o,
                         const void* dout, const float* lse, float* stats, float* dq_acc,
                         void* stream);

/* LAO backward of one hop: dq_acc += scale dS K (TL over n_q, fp32 atomics for
 * bf16); the visiting block's dK/dV contributions (TL over n_k) are written to
 * dk_acc/dv_acc, or added to them when accumulate != 0.  `stats` comes from
 * burst_bwd_preprocess on the pinned query block. */
BURST_API int burst_lao_bwd(const burst_hop* hop, const void* q, const void* k, const void* v,
                  const void* dout, const float* stats, float* dq_acc, float* dk_acc,
                  float* dv_acc, int accumulate, void* stream);

/* dq = dq_acc; dk = sum of nparts (1..16) dk partials; dv likewise (TL f32 -> dtype).
 * Outputs are checked for non-finite values (flags bit 1). */
BURST_API int burst_bwd_finalize(int dtype, int batch, int heads, int head_dim, int64_t n,
                       const float* dq_acc, const float* const* dk_parts,
                       const float* const* dv_parts, int nparts, void* dq, void* dk, void* dv,
                       int32_t* flags, void* stream);

/* out = sum of nparts TL f32 buffers (TL f32 -> dtype [batch, n, heads, head_dim]).
 * Assembles a gradient from per-hop contributions: the dQ contributions of the
 * reference's travelling-query backward payload (ring.py:65-83, 221-242; sim._collect
 * sim.py:450-471) when K/V/dK/dV stay pinned. */
BURST_API int burst_tl_sum(int dtype, int batch, int heads, int head_dim, int64_t n,
                 const float* const* parts, int nparts, void* out, int32_t* flags,
                 void* stream);

/* acc += part over one TL workspace of [batch, n, heads, head_dim] (both f32 TL).
 * Folds a received dK/dV (or dQ) contribution into the home accumulator as soon as
 * its exchange has landed, so a rank holds O(1) contribution buffers for any ring
 * size (the in-place accumulation of ring.backward_step, ring.py:239-241). */
BURST_API int burst_tl_accumulate(int batch, int heads, int head_dim, int64_t n, float* acc,
                        const float* part, void* stream);

/* Non-zero device-side flags raised by kernels since the last call (bit 0: a
 * row with no visible key, bit 1: non-finite output).  Synchronises `stream`. */
BURST_API int burst_read_flags(void* stream, int* flags_out);

/* Ring transport over NCCL (libnccl.so.2 resolved at run time).  The communicator is
 * non-blocking and watched: joining, and every posted exchange, must make progress
 * within `timeout_s` seconds, otherwise the communicator is aborted (stuck NCCL
 * kernels return) and this and every later call on the ring returns BURST_E_DEADLOCK
 * (DeadlockError, sim.py:290-310); an asynchronous NCCL error gives BURST_E_NCCL. */
BURST_API int burst_ring_unique_id(void* out_128_bytes);
BURST_API int burst_ring_create(const void* unique_id_128_bytes, int rank, int world, int device,
                      double timeout_s, void** ring);
/* Non-blocking health check: retires finished exchanges, reports how many were posted
 * and completed, and returns the ring's failure code (0 while healthy). */
BURST_API int burst_ring_poll(void* ring, uint64_t* posted, uint64_t* completed);
/* Block until every posted exchange has completed on the device, or the ring fails. */
BURST_API int burst_ring_wait(void* ring);
/* Grouped send(send_to) + recv(recv_from) of `bytes` on `stream`. */
BURST_API int burst_ring_exchange(void* ring, const void* send, void* recv, size_t bytes, int send_to,
                        int recv_from, void* stream);
/* One grouped exchange of several sends/receives (K/V rotation plus the dK/dV
 * contribution sent to its home rank) on `stream`. */
typedef struct {
  void* buf;
  size_t bytes;
  int32_t peer;
  int32_t is_send;
} burst_p2p;
BURST_API int burst_ring_sendrecv(void* ring, const burst_p2p* ops, int nops, void* stream);
BURST_API int burst_ring_destroy(void* ring);

/* Zero-SM ring transport (copy engines + CUDA IPC, ring.IpcTransport): the CUDA
 * runtime pieces of a mailbox exchange.  Handles are opaque byte blobs of
 * burst_ipc_handle_bytes() bytes (mem and event handles have the same size). */
BURST_API size_t burst_ipc_handle_bytes(void);
/* Dedicated, zeroed device allocation for a mailbox or flag array (an IPC handle
 * names a whole allocation). */
BURST_API int burst_ipc_alloc(size_t bytes, void** dev_ptr);
BURST_API int burst_ipc_free(void* dev_ptr);
BURST_API int burst_ipc_mem_handle(void* dev_ptr, void* out_handle);
BURST_API int burst_ipc_open_mem(const void* handle, void** dev_ptr);
BURST_API int burst_ipc_close_mem(void* dev_ptr);
/* Interprocess event (timing disabled); its handle opens in another process. */
BURST_API int burst_ipc_event_create(void** event, void* out_handle);
BURST_API int burst_ipc_event_open(const void* handle, void** event);
/* Device-side sequence flags of the IPC ring (no host round trip per exchange):
 * burst_signal_u32 writes `value` into the local staging word `stage`, then copies
 * it into `flag` (which may be IPC-mapped peer memory), both ordered after earlier
 * work of `stream`; burst_wait_u32 blocks `stream` until the local `flag` reaches
 * `value` (wrap-safe >=). */
BURST_API int burst_signal_u32(void* stream, void* flag, void* stage, uint32_t value);
BURST_API int burst_wait_u32(void* stream, void* flag, uint32_t value);
/* The IPC ring's exchange engine (ring.IpcTransport): flags/stage are this rank's
 * flag arrays ([world][2 slots][ready, free] uint32, zeroed), set_peer records the
 * IPC-mapped flag array and mailbox of every peer, set_mailbox this rank's mailbox
 * (2 slots of `slot_bytes`, split into tag regions of caps[0..2] bytes).  One
 * exchange call: free-signal every sender, wait each receiver's free flag, push the
 * SEND payloads into its slot regions (copy engines) and signal ready, wait every
 * sender's ready flag, copy out the receives that are not already the mailbox
 * region itself.  All ordered on `stream`; nothing blocks the host. */
typedef struct {
  void* buf;
  size_t bytes;
  int32_t peer;
  int32_t is_send;
  int32_t tag;       /* 0 rotating payload, 1 contribution, 2 exchange header */
  int32_t pad_;
} burst_ipc_op;
BURST_API int burst_ipc_ring_create(int rank, int world, void* flags, void* stage, void** out);
BURST_API int burst_ipc_ring_set_peer(void* ring, int peer, void* peer_flags, void* peer_mail);
BURST_API int burst_ipc_ring_set_mailbox(void* ring, void* mail, size_t slot_bytes,
                                         const uint64_t* caps);
BURST_API int burst_ipc_ring_exchange(void* ring, const burst_ipc_op* ops, int nops, void* stream);
BURST_API int burst_ipc_ring_destroy(void* ring);
BURST_API int burst_event_record(void* event, void* stream);
BURST_API int burst_stream_wait_event(void* stream, void* event);
BURST_API int burst_event_destroy(void* event);
/* Device-to-device (or peer) copy on `stream`, executed by the copy engines. */
BURST_API int burst_copy_async(void* dst, const void* src, size_t bytes, void* stream);

BURST_API const char* burst_last_error(void);
BURST_API int burst_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BURST_B200_H */
