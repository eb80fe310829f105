"""Ring engine: the per-rank hop loop of BurstAttention (GAO) with overlap.

Reference: the lockstep / threaded executors of sim.run_ring_pass
(sim.py:501-657): G rounds; at round r device i holds the payload of origin
(i - r) mod G; payloads move i -> i+1 through double buffers
(DoubleBuffer, sim.py:316-332).  Here one process (or thread) drives one rank:

forward, hop h:   comm stream:    send K/V(h) -> rank+1, recv K/V(h+1) <- rank-1
                  compute stream: LAO-fwd(q, K/V(h)) merged into (O_acc, m, l)
backward, hop h:  comm stream:    K/V rotation as above, plus the dK/dV
                                  contribution of hop h-1 sent to its home rank
                                  (one hop behind, so it overlaps hop h)
                  compute stream: LAO-bwd(q, dO, K/V(h)) -> dQ (pinned, fp32
                                  atomics) and dK/dV(h) contribution
                  end:            dK/dV = own + received contributions
The compute stream only waits for a transfer right before the hop that
consumes it, so every transfer except the last one overlaps a hop's kernel.

Transports:
  NcclTransport        one NCCL communicator via the C ABI (burst_ring_*); GPU
  LoopbackTransport    G ranks as threads in one process (the reference's
                       threaded executor); single-GPU simulation of a ring
  IpcTransport         copy-engine pushes into CUDA-IPC mailboxes (zero SM, f1)
  TorchDistTransport   torch.distributed P2P (gloo on CPU for host-logic tests)
"""

from __future__ import annotations

import ctypes
import threading
from collections import defaultdict
from typing import Sequence

import torch

from . import _lib
from .errors import DeadlockError, RingDesyncError
from .schedule import contributor_to, plan_hop

SEND, RECV = "send", "recv"

# ---------------------------------------------------------------------------
# streams
# ---------------------------------------------------------------------------

_tls = threading.local()


def comm_stream(device: torch.device):
    """Per-thread, per-device high-priority communication stream."""
    cache = getattr(_tls, "streams", None)
    if cache is None:
        cache = _tls.streams = {}
    key = device.index if device.index is not None else torch.cuda.current_device()
    if key not in cache:
        cache[key] = torch.cuda.Stream(device=key, priority=-1)
    return cache[key]


class _Streams:
    """Compute stream = caller's current stream; comm stream = side stream.
    On CPU tensors (host-logic tests) everything is synchronous."""

    def __init__(self, device: torch.device):
        self.cuda = device.type == "cuda"
        if self.cuda:
            self.compute = torch.cuda.current_stream(device)
            self.comm = comm_stream(device)
        else:
            self.compute = self.comm = None

    def comm_after_compute(self):
        if self.cuda:
            self.comm.wait_stream(self.compute)

    def compute_mark(self):
        """Event at the compute stream's current tail (None on CPU)."""
        if not self.cuda:
            return None
        ev = torch.cuda.Event()
        ev.record(self.compute)
        return ev

    def comm_wait(self, ev):
        if ev is not None:
            self.comm.wait_event(ev)

    def compute_after_comm(self):
        if self.cuda:
            self.compute.wait_stream(self.comm)


# ---------------------------------------------------------------------------
# transports
# ---------------------------------------------------------------------------

class _TransportBase:
    """Pass bookkeeping shared by the transports: `pass_seq` numbers this rank's passes
    (every rank runs the same passes in the same order, like the reference's lockstep
    rounds) and `finish` is the end-of-pass health check of the channel."""

    pass_seq = 0

    def next_pass(self) -> int:
        self.pass_seq = (self.pass_seq + 1) % (1 << 30)
        return self.pass_seq

    def finish(self, check: str) -> None:
        """Raise DeadlockError / NcclError for a failed channel ("sync": after waiting
        for every posted exchange; "async": only what is already known)."""


class SoloTransport(_TransportBase):
    rank, world = 0, 1

    def sendrecv(self, ops, stream):
        if ops:
            raise RingDesyncError("a world of one rank has nobody to exchange with")


def ring_timeout_s() -> float:
    """Progress horizon of a ring (DeadlockError after this long without any exchange
    completing; BURST_RING_TIMEOUT_S, default 600 s)."""
    import os
    return float(os.environ.get("BURST_RING_TIMEOUT_S", "600"))


class NcclTransport(_TransportBase):
    """NCCL communicator owned by libburst_b200.so (burst_ring_create): non-blocking,
    watched by a per-ring thread that aborts it when no exchange makes progress within
    `timeout_s` (DeadlockError, sim.py:290-310) or NCCL reports an asynchronous error."""

    def __init__(self, group=None, device: torch.device | None = None,
                 timeout_s: float | None = None):
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        uid = (ctypes.c_char * 128)()
        if self.rank == 0:
            _lib.call("burst_ring_unique_id", uid)
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0,
                                   group=group)
        uid = (ctypes.c_char * 128).from_buffer_copy(obj[0])
        handle = ctypes.c_void_p()
        self.timeout_s = float(timeout_s if timeout_s is not None else ring_timeout_s())
        _lib.call("burst_ring_create", uid, self.rank, self.world, dev.index,
                  ctypes.c_double(self.timeout_s), ctypes.byref(handle))
        self.handle = handle

    def finish(self, check: str) -> None:
        if check == "sync":
            _lib.call("burst_ring_wait", self.handle)
        elif check == "async":
            _lib.call("burst_ring_poll", self.handle, None, None)

    def progress(self) -> tuple[int, int]:
        """(exchanges posted, exchanges completed) so far on this ring."""
        a, b = ctypes.c_uint64(0), ctypes.c_uint64(0)
        _lib.call("burst_ring_poll", self.handle, ctypes.byref(a), ctypes.byref(b))
        return a.value, b.value

    def sendrecv(self, ops, stream):
        arr = (_lib.P2POp * len(ops))()
        for i, (kind, t, peer) in enumerate(ops):
            arr[i].buf = t.data_ptr()
            arr[i].bytes = t.numel() * t.element_size()
            arr[i].peer = peer
            arr[i].is_send = 1 if kind == SEND else 0
        _lib.call("burst_ring_sendrecv", self.handle, arr, len(ops),
                  ctypes.c_void_p(stream.cuda_stream))

    def close(self):
        if getattr(self, "handle", None):
            _lib.load().burst_ring_destroy(self.handle)
            self.handle = None


class IpcTransport(_TransportBase):
    """Zero-SM transport: each send is a copy-engine
    cudaMemcpyAsync into the receiver's CUDA-IPC mailbox (NVLink for peers on other
    GPUs), ordered by interprocess CUDA events; no SM is used, so the transfers
    never compete with the full-grid LAO kernels the way NCCL send/recv kernels do.

    Per exchange (all ranks call it in lockstep, like the reference's rounds,
    sim.py:551-574), with mailbox slot s alternating 0/1 (the DoubleBuffer of
    sim.py:316-332):
      1. capacity: every rank announces the bytes it will receive from each peer;
         a mailbox too small is reallocated and its IPC handle re-shared
         (all_gather_object; also the barrier that orders step 2 after the
         receivers' step-4 records of two exchanges ago);
      2. sender: comm stream waits the receiver's consumed[s] event, copies its
         SEND tensors back to back into the receiver's mailbox[from me][s], then
         records its own ready[s];
      3. barrier (every ready[s] recorded before anyone waits on it);
      4. receiver: waits the sender's ready[s], copies mailbox -> RECV tensors in
         the same order, records consumed[s].
    Host-side handshakes use `group` (gloo is enough).
    """

    def __init__(self, group=None, device: torch.device | None = None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        lib = _lib.load()
        self.hbytes = int(lib.burst_ipc_handle_bytes())
        self.slot = 0
        self.boxes = {}          # (src, slot) -> (device pointer, capacity): my mailboxes
        self.peer_box = {}       # (dst, slot) -> (device pointer, capacity) in dst's memory
        self.ready, self.consumed = [], []
        handles = []
        for _ in range(2):
            for lst in (self.ready, self.consumed):
                ev, h = ctypes.c_void_p(), (ctypes.c_char * self.hbytes)()
                _lib.call("burst_ipc_event_create", ctypes.byref(ev), h)
                lst.append(ev)
                handles.append(bytes(h))
        allh = [None] * self.world
        dist.all_gather_object(allh, handles, group=group)
        self.peer_ready, self.peer_consumed = {}, {}
        for r, hs in enumerate(allh):
            if r == self.rank:
                continue
            for s in range(2):
                for key, idx in ((self.peer_ready, 2 * s), (self.peer_consumed, 2 * s + 1)):
                    ev = ctypes.c_void_p()
                    buf = (ctypes.c_char * self.hbytes).from_buffer_copy(hs[idx])
                    _lib.call("burst_ipc_event_open", buf, ctypes.byref(ev))
                    key[(r, s)] = ev
        self.started = set()     # slots whose consumed event has been recorded once
        self.retired = []        # outgrown mailboxes (freed in close())

    def _grow(self, needs: dict, s: int) -> dict:
        """Reallocate my mailboxes that are too small; return {src: handle bytes}."""
        out = {}
        for src, nbytes in needs.items():
            box = self.boxes.get((src, s))
            if box is None or box[1] < nbytes:
                cap = max(nbytes, 2 * box[1] if box is not None else 0)
                if box is not None:   # the peer may still map it: freed in close()
                    self.retired.append(box[0])
                ptr = ctypes.c_void_p()
                _lib.call("burst_ipc_alloc", cap, ctypes.byref(ptr))
                self.boxes[(src, s)] = (ptr.value, cap)
                h = (ctypes.c_char * self.hbytes)()
                _lib.call("burst_ipc_mem_handle", ptr, h)
                out[src] = (bytes(h), cap)
        return out

    def sendrecv(self, ops, stream):
        d, s = self.dist, self.slot
        self.slot ^= 1
        sh = ctypes.c_void_p(stream.cuda_stream)
        needs = defaultdict(int)
        for kind, t, peer in ops:
            if kind == RECV:
                needs[peer] += t.numel() * t.element_size()
        # 1. capacity / handle exchange (+ the barrier of the protocol)
        new = self._grow(needs, s)
        allnew = [None] * self.world
        d.all_gather_object(allnew, new, group=self.group)
        for r, m in enumerate(allnew):
            if r != self.rank and self.rank in m:
                h, cap = m[self.rank]
                old = self.peer_box.get((r, s))
                if old is not None:
                    _lib.call("burst_ipc_close_mem", ctypes.c_void_p(old[0]))
                ptr = ctypes.c_void_p()
                buf = (ctypes.c_char * self.hbytes).from_buffer_copy(h)
                _lib.call("burst_ipc_open_mem", buf, ctypes.byref(ptr))
                self.peer_box[(r, s)] = (ptr.value, cap)
        # 2. pushes into the receivers' mailboxes (copy engines)
        offs = defaultdict(int)
        waited = set()
        for kind, t, peer in ops:
            if kind != SEND:
                continue
            if s in self.started and peer not in waited:
                _lib.call("burst_stream_wait_event", sh, self.peer_consumed[(peer, s)])
                waited.add(peer)
            ptr, cap = self.peer_box[(peer, s)]
            nb = t.numel() * t.element_size()
            if offs[peer] + nb > cap:
                raise RingDesyncError(f"rank {self.rank}: payload to {peer} exceeds its mailbox")
            _lib.call("burst_copy_async", ctypes.c_void_p(ptr + offs[peer]),
                      ctypes.c_void_p(t.data_ptr()), nb, sh)
            offs[peer] += nb
        _lib.call("burst_event_record", self.ready[s], sh)
        # 3. every ready[s] recorded before anyone waits on it
        d.barrier(group=self.group)
        # 4. mailbox -> destination tensors
        offs = defaultdict(int)
        waited = set()
        for kind, t, peer in ops:
            if kind != RECV:
                continue
            if peer not in waited:
                _lib.call("burst_stream_wait_event", sh, self.peer_ready[(peer, s)])
                waited.add(peer)
            box = self.boxes[(peer, s)][0]
            nb = t.numel() * t.element_size()
            _lib.call("burst_copy_async", ctypes.c_void_p(t.data_ptr()),
                      ctypes.c_void_p(box + offs[peer]), nb, sh)
            offs[peer] += nb
        _lib.call("burst_event_record", self.consumed[s], sh)
        self.started.add(s)

    def close(self):
        lib = _lib.load()
        torch.cuda.synchronize(self.device)
        for ptr, _ in self.peer_box.values():
            lib.burst_ipc_close_mem(ctypes.c_void_p(ptr))
        self.peer_box = {}
        self.dist.barrier(group=self.group)     # every peer unmapped before freeing
        for ptr in [p for p, _ in self.boxes.values()] + self.retired:
            lib.burst_ipc_free(ctypes.c_void_p(ptr))
        self.boxes, self.retired = {}, []


class TorchDistTransport(_TransportBase):
    """torch.distributed P2P (gloo on CPU: the multi-process host-logic tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def _global(self, peer):
        return self.dist.get_global_rank(self.group, peer) if self.group is not None else peer

    def sendrecv(self, ops, stream):
        d = self.dist
        p2p = [d.P2POp(d.isend if kind == SEND else d.irecv, t, self._global(peer), self.group)
               for kind, t, peer in ops]
        if not p2p:
            return
        ctx = torch.cuda.stream(stream) if stream is not None else _nullctx()
        with ctx:
            for req in d.batch_isend_irecv(p2p):
                req.wait()


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


class LoopbackHub:
    """Mailboxes + barrier shared by the G rank-threads of one process."""

    def __init__(self, world: int, timeout: float = 120.0):
        self.world = world
        self.barrier = threading.Barrier(world, timeout=timeout)
        self.lock = threading.Lock()
        self.box = defaultdict(list)    # (seq, src, dst) -> [(tensor, event)]
        self.copied = defaultdict(list)  # (seq, src) -> [events of finished copies]

    def transport(self, rank: int) -> "LoopbackTransport":
        return LoopbackTransport(self, rank)


class LoopbackTransport(_TransportBase):
    """One rank of a LoopbackHub: device-to-device copies on the comm stream,
    ordered with CUDA events exactly like a real send/recv (RingChannel,
    sim.py:281-313; DeadlockError on a stalled peer, sim.py:290-310)."""

    def __init__(self, hub: LoopbackHub, rank: int):
        self.hub, self.rank, self.world = hub, rank, hub.world
        self.seq = 0

    def _sync(self):
        try:
            self.hub.barrier.wait()
        except threading.BrokenBarrierError as e:
            raise DeadlockError(f"rank {self.rank}: ring peer did not arrive") from e

    def sendrecv(self, ops, stream):
        hub, seq = self.hub, self.seq
        self.seq += 1
        cuda = stream is not None
        with hub.lock:
            for kind, t, peer in ops:
                if kind == SEND:
                    ev = None
                    if cuda:
                        ev = torch.cuda.Event()
                        ev.record(stream)
                    hub.box[(seq, self.rank, peer)].append((t, ev))
        self._sync()
        taken = defaultdict(int)
        for kind, t, peer in ops:
            if kind != RECV:
                continue
            with hub.lock:
                items = hub.box.get((seq, peer, self.rank), [])
                if taken[peer] >= len(items):
                    raise RingDesyncError(f"rank {self.rank}: no payload from {peer} (seq {seq})")
                src, ev = items[taken[peer]]
            taken[peer] += 1
            if src.shape != t.shape or src.dtype != t.dtype:
                raise RingDesyncError(f"rank {self.rank}: payload from {peer} is "
                                      f"{tuple(src.shape)}/{src.dtype}, expected "
                                      f"{tuple(t.shape)}/{t.dtype}")
            if cuda:
                stream.wait_event(ev)
                with torch.cuda.stream(stream):
                    t.copy_(src, non_blocking=True)
                done = torch.cuda.Event()
                done.record(stream)
            else:
                t.copy_(src)
                done = None
            with hub.lock:
                hub.copied[(seq, peer)].append(done)
        self._sync()
        if cuda:
            # the sender may reuse its buffers only after every receiver copied
            for ev in hub.copied.get((seq, self.rank), []):
                stream.wait_event(ev)
        self._sync()
        with hub.lock:
            for dst in range(self.world):
                hub.box.pop((seq, self.rank, dst), None)
            hub.copied.pop((seq, self.rank), None)


# ---------------------------------------------------------------------------
# the hop loops
# ---------------------------------------------------------------------------

class SlotLog:
    """Exchange headers of one pass: the reference's desync checks (RingDesyncError on
    an unexpected payload count, origin or sequence, sim.py:570-574 and 622-631) on a
    real ring.  In every exchange slot rank r also sends [pass, slot, r, origin] to
    r+1 -- origin = the rank whose block the slot's rotating payload carries, -1 when
    the slot rotates nothing -- and receives its predecessor's header into row `slot`
    of a device log.  At pass end the log is compared with what the schedule implies,
    so a rank that skipped, repeated or reordered an exchange, ran another pass, or
    forwarded a block from the wrong origin raises RingDesyncError."""

    def __init__(self, transport, device: torch.device, slots, origin_fn):
        import numpy as np
        G, r = transport.world, transport.rank
        self.active = G > 1
        if not self.active:
            return
        self.G, self.r = G, r
        self.row = {slot: i for i, slot in enumerate(slots)}
        pid = transport.next_pass()
        mine = np.array([[pid, sl, r, origin_fn(r, sl)] for sl in slots], dtype=np.int32)
        prev = (r - 1) % G
        self.expected = np.array([[pid, sl, prev, origin_fn(prev, sl)] for sl in slots],
                                 dtype=np.int32)
        t = torch.from_numpy(mine)
        if device.type == "cuda":
            t = t.pin_memory().to(device, non_blocking=True)
        self.send = t
        self.log = torch.full((len(slots), 4), -2, dtype=torch.int32, device=device)
        self.device = device

    def ops(self, slot: int):
        if not self.active:
            return []
        i = self.row[slot]
        return [(SEND, self.send[i], (self.r + 1) % self.G),
                (RECV, self.log[i], (self.r - 1) % self.G)]

    def _check(self, got) -> None:
        got = got.numpy() if hasattr(got, "numpy") else got
        for i in range(len(self.expected)):
            if tuple(got[i]) != tuple(self.expected[i]):
                raise RingDesyncError(
                    f"rank {self.r}: exchange slot {int(self.expected[i][1])} delivered header "
                    f"(pass, slot, sender, origin) = {tuple(int(x) for x in got[i])}, expected "
                    f"{tuple(int(x) for x in self.expected[i])}")

    def finish(self, check: str, stream) -> None:
        if not self.active or check == "off":
            return
        if self.device.type != "cuda" or check == "sync":
            if stream is not None:
                stream.synchronize()
            self._check(self.log.cpu())
        else:
            from .kernels import PENDING
            PENDING.add_check(self.log, stream, self._check)


def _rotating(G: int):
    """origin_fn of a pass whose payload rotates at slots h < G-1 (K/V, or Q/dO)."""
    return lambda rank, h: (rank - h) % G if h < G - 1 else -1


def backward_slots(G: int) -> list:
    """Exchange slots of a backward pass: K/V rotation at h < G-1, contribution
    homecoming (one hop late) at h >= 2, and the final homecoming slot G."""
    return [h for h in range(G) if h < G - 1 or h >= 2] + ([G] if G > 1 else [])


def ring_forward(q, k, v, scale: float, causal: bool, zigzag: bool, transport, kernels,
                 n_valid: int | None = None, recorder=None, grid=None, check: str = "sync"):
    """One rank's forward pass.  Returns (O [B,n,H,D], lse [B,H,n] natural log).
    `n_valid`: real global length when the shards are zero-padded (reference pad=True).
    `recorder`: optional trace.PassRecorder (measured timeline + ledger, sim.py:118-261).
    `grid`: optional masks.GridMask bound to the global length (BlockGrid).
    `check`: when the pass's device error word is read ("sync" | "async" | "off",
    kernels.finish; MaskError / NonFiniteError as in PartialAttn.finalize)."""
    B, n, H, D = q.shape
    G, r = transport.world, transport.rank
    S = _Streams(q.device)
    o = torch.empty_like(q)
    lse = torch.empty(B, H, n, dtype=torch.float32, device=q.device)
    state = kernels.fwd_state(q, running=G > 1)
    slog = SlotLog(transport, q.device, list(range(G - 1)), _rotating(G))
    cur_k, cur_v = k, v
    spare = None
    finalized = False
    computed = False             # a hop has merged into the running state
    prev = S.compute_mark()      # compute tail before hop h (buffers it still reads)
    for h in range(G):
        plan = plan_hop(r, G, h, n, causal, zigzag, n_valid, grid)
        exchanged = False
        # launch the hop's kernel first, then post the transfer on the comm stream:
        # both run concurrently (the comm waits only for the PREVIOUS hop's kernel,
        # which last read the buffer being received into)
        if recorder is not None:
            recorder.mark(h, "compute_start", S.compute)
        if not plan.skip:
            fin = h == G - 1 and plan.covers_all_queries(n)
            kernels.fwd(plan, q, cur_k, cur_v, scale, state, o, lse, first=not computed,
                        finalize=fin, stream=S.compute)
            finalized = finalized or fin
            computed = True
        if recorder is not None:
            recorder.mark(h, "compute_end", S.compute)
        done = S.compute_mark()
        if h < G - 1:
            if spare is None:
                spare = (torch.empty_like(k), torch.empty_like(v))
            S.comm_wait(prev)
            ops = [(SEND, cur_k, (r + 1) % G), (SEND, cur_v, (r + 1) % G),
                   (RECV, spare[0], (r - 1) % G), (RECV, spare[1], (r - 1) % G)]
            if recorder is not None:
                recorder.count_send("forward", ops)
                recorder.mark(h, "send_start", S.comm)
            transport.sendrecv(ops + slog.ops(h), S.comm)
            if recorder is not None:
                recorder.mark(h, "send_end", S.comm)
                recorder.mark(h, "recv_ready", S.comm)
            exchanged = True
        prev = done
        if exchanged:
            S.compute_after_comm()
            (cur_k, cur_v), spare = spare, (cur_k, cur_v)
            if spare[0] is k:
                spare = None   # never receive into the caller's tensors
    if not finalized:
        kernels.fwd_finalize(state, o, lse, stream=S.compute)
    kernels.finish(state, check, stream=S.compute)
    slog.finish(check, S.compute)
    transport.finish(check)
    return o, lse


def split_own_hop(plan, n: int, world: int):
    """(first, last) query-row halves of the own-block hop: `first` runs at hop 0 and
    `last` after hop G-1, where it overlaps the final homecoming exchange (the
    contribution of hop G-1 going home), which otherwise has no kernel to hide
    behind (the one-hop lag of sim.py:19-21).  The later half holds the larger
    share of a causal block (its queries see every earlier key), and the split row
    is a multiple of 128 so both halves keep the tile-aligned backward kernel.
    Returns (plan, None) when there is nothing to overlap (G == 1) or no aligned split."""
    if world == 1 or plan.skip or plan.q_begin != 0 or plan.q_len != n:
        return plan, None
    cut = (n // 2) // 128 * 128
    if cut == 0:
        return plan, None
    from dataclasses import replace
    return replace(plan, q_len=cut), replace(plan, q_begin=cut, q_len=n - cut)


def _part_exchange(r: int, G: int, n: int, causal: bool, zigzag: bool, hop: int, send_bufs,
                   recv_bufs, n_valid=None, grid=None):
    """Ops moving the dK/dV contribution computed at `hop` to its home rank, and
    receiving into `recv_bufs` the one computed for ours.  Returns (ops, received?)."""
    ops = []
    mine = plan_hop(r, G, hop, n, causal, zigzag, n_valid, grid)
    if not mine.skip:
        ops += [(SEND, send_bufs[0], mine.src), (SEND, send_bufs[1], mine.src)]
    c = contributor_to(r, G, hop)
    theirs = plan_hop(c, G, hop, n, causal, zigzag, n_valid, grid)
    if not theirs.skip:
        ops += [(RECV, recv_bufs[0], c), (RECV, recv_bufs[1], c)]
    return ops, not theirs.skip


def ring_backward(q, k, v, o, lse, dout, scale: float, causal: bool, zigzag: bool, transport,
                  kernels, n_valid: int | None = None, recorder=None, grid=None,
                  check: str = "sync"):
    """One rank's backward pass.  Returns (dq, dk, dv) in q's dtype.

    Contribution buffers are O(1) in the ring size: `own` accumulates this rank's
    dK/dV, `send[2]` hold the contributions of the last two hops (each goes home one
    hop later), `recv` the contribution arriving for our block, folded into `own`
    (burst_tl_accumulate) before the next hop -- the in-place accumulation of
    ring.backward_step (ring.py:239-241).  The own block is computed in two query
    halves (split_own_hop) so the final homecoming exchange overlaps a kernel.
    `recorder`: optional trace.PassRecorder (see ring_forward)."""
    B, n, H, D = q.shape
    G, r = transport.world, transport.rank
    S = _Streams(q.device)
    st = kernels.bwd_prepare(o, dout, lse, stream=S.compute)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    own = (kernels.part(k), kernels.part(v))
    slog = SlotLog(transport, q.device, backward_slots(G), _rotating(G))
    send = [None, None]
    recv = (kernels.part(k), kernels.part(v)) if G > 1 else None
    pending = False              # `recv` holds a contribution not yet folded into `own`
    own_last = None              # second query half of the own block (after hop G-1)
    cur_k, cur_v = k, v
    spare = None
    for h in range(G):
        plan = plan_hop(r, G, h, n, causal, zigzag, n_valid, grid)
        if h == 0:
            plan, own_last = split_own_hop(plan, n, G)
        if recorder is not None:
            recorder.mark(h, "compute_start", S.compute)
        if pending:              # landed in the previous slot (compute waited for it)
            kernels.accumulate(own, recv, k, stream=S.compute)
            pending = False
        # this slot's transfers wait for everything above: hop h-1's kernel (it made
        # the contribution sent now and last read `spare`) and the fold of `recv`
        ready = S.compute_mark()
        if h == 0:
            target = own
        else:
            if send[h % 2] is None:
                send[h % 2] = (kernels.part(k), kernels.part(v))
            target = send[h % 2]
        if not plan.skip:
            kernels.bwd(plan, q, cur_k, cur_v, dout, scale, st, target[0], target[1],
                        accumulate=False, stream=S.compute)
        elif h == 0:                  # own block fully masked (grid): no contribution
            kernels.zero_(target, stream=S.compute)
        if recorder is not None:
            recorder.mark(h, "compute_end", S.compute)
        ops = []
        if h < G - 1:
            if spare is None:
                spare = (torch.empty_like(k), torch.empty_like(v))
            ops += [(SEND, cur_k, (r + 1) % G), (SEND, cur_v, (r + 1) % G),
                    (RECV, spare[0], (r - 1) % G), (RECV, spare[1], (r - 1) % G)]
        if h >= 2:
            p_ops, got = _part_exchange(r, G, n, causal, zigzag, h - 1, send[(h - 1) % 2],
                                        recv, n_valid, grid)
            ops += p_ops
            pending = got
        # every rank takes part in every exchange slot (a slot depends only on
        # h and G), even with no op of its own: keeps loopback/collective
        # transports in lockstep when causal hops are skipped
        slot = h < G - 1 or h >= 2
        if slot:
            S.comm_wait(ready)
            if recorder is not None:
                recorder.count_send("backward", ops)
                recorder.mark(h, "send_start", S.comm)
            transport.sendrecv(ops + slog.ops(h), S.comm)
            if recorder is not None:
                recorder.mark(h, "send_end", S.comm)
                recorder.mark(h, "recv_ready", S.comm)
            S.compute_after_comm()
        if h < G - 1:
            (cur_k, cur_v), spare = spare, (cur_k, cur_v)
            if spare[0] is k:
                spare = None
    parts_k, parts_v = [own[0]], [own[1]]
    if G > 1:
        # homecoming of hop G-1's contribution, overlapped by the own block's last half
        if recorder is not None:
            recorder.mark(G, "compute_start", S.compute)
        if pending:
            kernels.accumulate(own, recv, k, stream=S.compute)
        ready = S.compute_mark()
        p_ops, got = _part_exchange(r, G, n, causal, zigzag, G - 1, send[(G - 1) % 2], recv,
                                    n_valid, grid)
        S.comm_wait(ready)
        if recorder is not None:
            recorder.count_send("backward", p_ops)
            recorder.mark(G, "send_start", S.comm)
        transport.sendrecv(p_ops + slog.ops(G), S.comm)
        if recorder is not None:
            recorder.mark(G, "send_end", S.comm)
            recorder.mark(G, "recv_ready", S.comm)
        if own_last is not None:
            kernels.bwd(own_last, q, k, v, dout, scale, st, own[0], own[1], accumulate=True,
                        stream=S.compute)
        if recorder is not None:
            recorder.mark(G, "compute_end", S.compute)
        S.compute_after_comm()
        if got:
            parts_k.append(recv[0])
            parts_v.append(recv[1])
    kernels.bwd_finalize(st, parts_k, parts_v, dq, dk, dv, stream=S.compute)
    kernels.finish(st, check, stream=S.compute)
    slog.finish(check, S.compute)
    transport.finish(check)
    return dq, dk, dv


def _qpart_exchange(r: int, G: int, n: int, causal: bool, zigzag: bool, hop: int, send_buf,
                    recv_buf, n_valid=None, grid=None):
    """Ops moving the dQ contribution computed at `hop` (for the visiting query
    block) to that block's home rank, and receiving into `recv_buf` the one
    computed for ours.  Returns (ops, received?)."""
    ops = []
    src = (r - hop) % G                        # origin of the query block I processed
    if not plan_hop(src, G, (src - r) % G, n, causal, zigzag, n_valid, grid).skip:
        ops.append((SEND, send_buf, src))
    c = (r + hop) % G                          # the rank that processed MY block at `hop`
    got = not plan_hop(r, G, (r - c) % G, n, causal, zigzag, n_valid, grid).skip
    if got:
        ops.append((RECV, recv_buf, c))
    return ops, got


def ring_backward_qtravel(q, k, v, o, lse, dout, scale: float, causal: bool, zigzag: bool,
                          transport, kernels, n_valid: int | None = None, recorder=None,
                          grid=None, check: str = "sync"):
    """One rank's backward pass with the REFERENCE's payload:
    the query-side record (Q, dO, lse/D statistics) travels the ring and K/V/dK/dV
    stay pinned (BackwardBody ring.py:65-83, backward_step ring.py:221-242,
    Alg. 2 of the paper).  The reference also carries the dQ accumulator in the
    body; here each hop's dQ contribution goes home one hop later instead (the
    lag sim.py:19-21 says a real system needs), so no transfer waits on a kernel
    of the same hop, and is folded into the home dQ accumulator as soon as it
    lands (O(1) buffers).  The own block runs in two query halves like
    ring_backward, the second one overlapping the last dQ homecoming.  Wire bytes
    per hop: 2·n·H·D·elem (Q, dO) + statistics + an fp32 dQ contribution, vs K/V +
    fp32 dK/dV for ring_backward.  Returns (dq, dk, dv) in q's dtype."""
    B, n, H, D = q.shape
    G, r = transport.world, transport.rank
    S = _Streams(q.device)
    st = kernels.bwd_prepare(o, dout, lse, stream=S.compute)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    dk_acc, dv_acc = kernels.part(k), kernels.part(v)
    payload = [q, dout] + kernels.stats_tensors(st)      # the visiting query block
    slog = SlotLog(transport, q.device, backward_slots(G), _rotating(G))
    spare = None
    send = [None, None]
    recv = kernels.dq_recv(q) if G > 1 else None
    pending = False
    own_last = None
    first_kv = True
    for h in range(G):
        src = (r - h) % G
        plan = plan_hop(src, G, (src - r) % G, n, causal, zigzag, n_valid, grid)
        if h == 0:
            plan, own_last = split_own_hop(plan, n, G)
        if recorder is not None:
            recorder.mark(h, "compute_start", S.compute)
        if pending:
            kernels.accumulate_dq(st, recv, q, stream=S.compute)
            pending = False
        ready = S.compute_mark()
        if h == 0:
            vst = st                                     # own queries: own dQ accumulator
        else:
            # zeroed on the compute stream: the buffer was last read by slot h-1's
            # send, which the compute stream has waited for
            send[h % 2] = kernels.dq_part(q, stream=S.compute, reuse=send[h % 2])
            vst = kernels.visiting_state(st, payload[2:], send[h % 2])
        if not plan.skip:
            kernels.bwd(plan, payload[0], k, v, payload[1], scale, vst, dk_acc, dv_acc,
                        accumulate=not first_kv, stream=S.compute)
            first_kv = False
        if recorder is not None:
            recorder.mark(h, "compute_end", S.compute)
        ops = []
        if h < G - 1:
            if spare is None:
                spare = [torch.empty_like(t) for t in payload]
            ops += [(SEND, t, (r + 1) % G) for t in payload]
            ops += [(RECV, t, (r - 1) % G) for t in spare]
        if h >= 2:
            p_ops, got = _qpart_exchange(r, G, n, causal, zigzag, h - 1, send[(h - 1) % 2],
                                         recv, n_valid, grid)
            ops += p_ops
            pending = got
        slot = h < G - 1 or h >= 2
        if slot:
            S.comm_wait(ready)
            if recorder is not None:
                recorder.count_send("backward", ops)
                recorder.mark(h, "send_start", S.comm)
            transport.sendrecv(ops + slog.ops(h), S.comm)
            if recorder is not None:
                recorder.mark(h, "send_end", S.comm)
                recorder.mark(h, "recv_ready", S.comm)
            S.compute_after_comm()
        if h < G - 1:
            payload, spare = spare, payload
            if spare[0] is q:
                spare = None   # never receive into the caller's tensors
    got = False
    if G > 1:
        if recorder is not None:
            recorder.mark(G, "compute_start", S.compute)
        if pending:
            kernels.accumulate_dq(st, recv, q, stream=S.compute)
        ready = S.compute_mark()
        p_ops, got = _qpart_exchange(r, G, n, causal, zigzag, G - 1, send[(G - 1) % 2], recv,
                                     n_valid, grid)
        S.comm_wait(ready)
        if recorder is not None:
            recorder.count_send("backward", p_ops)
            recorder.mark(G, "send_start", S.comm)
        transport.sendrecv(p_ops + slog.ops(G), S.comm)
        if recorder is not None:
            recorder.mark(G, "send_end", S.comm)
            recorder.mark(G, "recv_ready", S.comm)
        if own_last is not None:
            kernels.bwd(own_last, q, k, v, dout, scale, st, dk_acc, dv_acc,
                        accumulate=not first_kv, stream=S.compute)
            first_kv = False
        if recorder is not None:
            recorder.mark(G, "compute_end", S.compute)
        S.compute_after_comm()
    if first_kv:                                  # every hop skipped: no key is visible
        kernels.zero_((dk_acc, dv_acc), stream=S.compute)
    kernels.bwd_finalize_qtravel(st, [recv] if got else [], dk_acc, dv_acc, dq, dk, dv,
                                 stream=S.compute)
    kernels.finish(st, check, stream=S.compute)
    slog.finish(check, S.compute)
    transport.finish(check)
    return dq, dk, dv


def ring_comm_bytes(n_local: int, batch: int, heads: int, d: int, world: int, elem: int,
                    causal: bool, zigzag: bool, rank: int = 0,
                    bwd_payload: str = "kv") -> tuple[int, int]:
    """Bytes `rank` sends per forward and per backward pass (the ledger of
    sim.py:118-153).  bwd_payload "kv": K/V + fp32 dK/dV contributions (this
    build's default); "q": Q, dO, lse/D statistics + fp32 dQ contributions (the
    reference's payload, ring_backward_qtravel)."""
    kv = 2 * batch * n_local * heads * d * elem
    nt = -(-n_local // 128) * 128
    fwd = (world - 1) * kv
    if bwd_payload == "q":
        stats = 2 * batch * heads * nt * 4
        qpart = batch * nt * heads * d * 4
        bwd = (world - 1) * (kv + stats)
        for h in range(1, world):
            src = (rank - h) % world
            if not plan_hop(src, world, (src - rank) % world, n_local, causal, zigzag).skip:
                bwd += qpart
        return fwd, bwd
    part = 2 * batch * nt * heads * d * 4
    bwd = (world - 1) * kv
    bwd += sum(part for h in range(1, world)
               if not plan_hop(rank, world, h, n_local, causal, zigzag).skip)
    return fwd, bwd


_loopback_streams: dict = {}   # (device, rank) -> (compute stream, {device: comm stream})
_loopback_lock = threading.Lock()


def _rank_streams(dev: int, rank: int):
    """Persistent streams of a loopback rank: repeated passes reuse the same
    streams (and so the caching allocator's per-stream pools)."""
    with _loopback_lock:
        key = (dev, rank)
        if key not in _loopback_streams:
            _loopback_streams[key] = (torch.cuda.Stream(device=dev),
                                      {dev: torch.cuda.Stream(device=dev, priority=-1)})
        return _loopback_streams[key]


def run_ranks(world: int, fn, timeout: float = 600.0,
              deadlock_timeout: float | None = None) -> Sequence:
    """Run fn(rank, transport) for `world` loopback ranks in threads (the
    reference's threaded executor, sim.py:575-620); re-raise the first error.
    `deadlock_timeout`: seconds a rank may wait for its peers at an exchange before
    the pass fails with DeadlockError (sim.py:290-310, 622-631)."""
    hub = LoopbackHub(world, timeout=deadlock_timeout if deadlock_timeout is not None else 120.0)
    out = [None] * world
    errors = []
    dev = torch.cuda.current_device() if torch.cuda.is_available() else None
    # the caller produced the shards on its own stream (asynchronously); the rank
    # streams are non-blocking, so they must wait for it before touching them
    caller = torch.cuda.current_stream(dev) if dev is not None else None

    def work(rank):
        try:
            if dev is not None:
                torch.cuda.set_device(dev)
                s, comm = _rank_streams(dev, rank)
                _tls.streams = comm
                s.wait_stream(caller)
                with torch.cuda.stream(s):
                    out[rank] = fn(rank, hub.transport(rank))
                s.synchronize()
            else:
                out[rank] = fn(rank, hub.transport(rank))
        except BaseException as e:  # noqa: BLE001 - surfaced below
            errors.append(e)
            hub.barrier.abort()

    threads = [threading.Thread(target=work, args=(i,), daemon=True) for i in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout)
    if errors:
        # the first rank to fail names the cause; peers report the broken barrier
        first = next((e for e in errors if not isinstance(e, DeadlockError)), errors[0])
        raise first
    if any(t.is_alive() for t in threads):
        raise DeadlockError("ring ranks failed to finish")
    return out
