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
# op tags (optional 4th element of an op): the region of a mailbox transport's slot
# the payload lands in (IpcTransport); other transports ignore them
TAG_ROT, TAG_PART, TAG_HDR = 0, 1, 2
HDR_BYTES = 16          # one SlotLog header: int32 [pass, slot, sender, origin]

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
    mailbox = False     # True: receives land in transport-owned buffers handed out by rx()

    def reserve(self, need: dict) -> None:
        """Receive capacity per op tag for the coming pass (mailbox transports)."""

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
        for i, (kind, t, peer, *_) in enumerate(ops):
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


class _DevBuf:
    """__cuda_array_interface__ over a raw device range (torch.as_tensor views it)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 2}


class IpcTransport(_TransportBase):
    """Zero-SM transport: each send is a copy-engine
    cudaMemcpyAsync straight into the receiver's CUDA-IPC mailbox (NVLink for peers
    on other GPUs); no SM is used, so transfers never compete with the full-grid LAO
    kernels the way NCCL send/recv kernels do, and no host round trip happens per
    exchange: ordering is carried by device-side sequence flags.

    Mailboxes: two slots (the DoubleBuffer of sim.py:316-332; exchange e uses slot
    e % 2), each split into per-tag regions -- 0: the rotating payload (K/V, or Q/dO/
    statistics), 1: a contribution going home, 2: exchange headers (SlotLog) -- sized
    once per shape by `reserve` (every rank calls it with the same, shape-derived
    sizes at pass start; only a growth is collective).  The ring engine receives IN
    PLACE: `rx` hands out views of the next exchange's slot and the kernels read
    them directly (no mailbox -> tensor copy).

    Exchange e, slot s, sequence q = e + 1, on the comm stream (which the engine has
    already ordered after the compute that last read slot s):
      1. for every peer p we receive from: flags_p[me][s].free = q (p may now
         overwrite our slot s);
      2. for every peer d we send to: wait flags_me[d][s].free >= q, push the SEND
         tensors into d's slot s regions, then flags_d[me][s].ready = q;
      3. for every peer p we receive from: wait flags_me[p][s].ready >= q.
    Waits are cuStreamWaitValue32 on our own memory; signals a staged 4-byte copy
    into the peer's flag array (burst_signal_u32).  A stalled peer stalls the comm
    stream; `finish("sync")` then reports DeadlockError after the ring timeout."""

    mailbox = True
    TAGS = (0, 1, 2)

    def __init__(self, group=None, device: torch.device | None = None,
                 timeout_s: float | None = None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.timeout_s = float(timeout_s if timeout_s is not None else ring_timeout_s())
        lib = _lib.load()
        self._exchange = lib.burst_ipc_ring_exchange
        self.hbytes = int(lib.burst_ipc_handle_bytes())
        self.e = 0                       # exchanges posted so far (all ranks in lockstep)
        self.caps = {t: 0 for t in self.TAGS}
        self.mail, self.slot_bytes = None, 0     # my mailbox: 2 slots
        self.peer_mail = {}              # peer -> base of its mailbox (IPC-mapped)
        self.retired = []                # outgrown mailboxes (freed in close())
        self.host_us = []                # host time to post each exchange (measurement)
        self.c_us = []                   # ... of which inside burst_ipc_ring_exchange
        # flags: [world][2 slots][ready, free] uint32 in my memory, written by peers;
        # stage: the same shape, local staging words of the signals I send
        n = self.world * 4 * 4
        fl, st = ctypes.c_void_p(), ctypes.c_void_p()
        _lib.call("burst_ipc_alloc", n, ctypes.byref(fl))
        _lib.call("burst_ipc_alloc", n, ctypes.byref(st))
        self.flags, self.stage = fl.value, st.value
        ring = ctypes.c_void_p()
        _lib.call("burst_ipc_ring_create", self.rank, self.world, fl, st, ctypes.byref(ring))
        self.ring = ring
        h = (ctypes.c_char * self.hbytes)()
        _lib.call("burst_ipc_mem_handle", fl, h)
        allh = [None] * self.world
        dist.all_gather_object(allh, bytes(h), group=group)
        self.peer_flags = {}
        for r, hb in enumerate(allh):
            if r != self.rank:
                self.peer_flags[r] = self._open(hb)
                _lib.call("burst_ipc_ring_set_peer", self.ring, r,
                          ctypes.c_void_p(self.peer_flags[r]), None)
        self.last_wait = None            # event after the newest exchange
        self._events = (torch.cuda.Event(), torch.cuda.Event())
        self._arr = (_lib.IpcOp * 16)()

    # ---------------------------------------------------------------- layout
    def _open(self, hb: bytes) -> int:
        ptr = ctypes.c_void_p()
        buf = (ctypes.c_char * self.hbytes).from_buffer_copy(hb)
        _lib.call("burst_ipc_open_mem", buf, ctypes.byref(ptr))
        return ptr.value

    def _off(self, tag: int) -> int:
        return sum(self.caps[t] for t in self.TAGS if t < tag)

    def reserve(self, need: dict) -> None:
        """Make every tag region hold at least need[tag] bytes.  Called by every rank at
        the same point of every pass with the same (shape-derived) sizes, so a growth
        -- collective: device sync, barrier, reallocation, handle exchange -- happens
        on all ranks together; otherwise this is a no-op."""
        grow = {t: max(self.caps[t], -(-int(need.get(t, 0)) // 256) * 256) for t in self.TAGS}
        if grow == self.caps and self.mail is not None:
            return
        torch.cuda.synchronize(self.device)
        d = self.dist
        d.barrier(group=self.group)            # no peer still pushes into the old slots
        for ptr in self.peer_mail.values():
            _lib.call("burst_ipc_close_mem", ctypes.c_void_p(ptr))
        self.peer_mail = {}
        if self.mail is not None:
            self.retired.append(self.mail)     # views may still reference it
        self.caps = grow
        self.slot_bytes = max(sum(grow.values()), 256)
        ptr = ctypes.c_void_p()
        _lib.call("burst_ipc_alloc", 2 * self.slot_bytes, ctypes.byref(ptr))
        self.mail = ptr.value
        caps = (ctypes.c_uint64 * 3)(*[grow[t] for t in self.TAGS])
        _lib.call("burst_ipc_ring_set_mailbox", self.ring, ptr, self.slot_bytes, caps)
        h = (ctypes.c_char * self.hbytes)()
        _lib.call("burst_ipc_mem_handle", ptr, h)
        allh = [None] * self.world
        d.all_gather_object(allh, bytes(h), group=self.group)
        for r, hb in enumerate(allh):
            if r != self.rank:
                self.peer_mail[r] = self._open(hb)
                _lib.call("burst_ipc_ring_set_peer", self.ring, r, None,
                          ctypes.c_void_p(self.peer_mail[r]))

    def rx(self, likes, tag: int) -> list:
        """Receive buffers of the NEXT exchange for `likes` (in op order): views of our
        mailbox slot, region `tag`; the pushes land there and the kernels read them."""
        if self.mail is None:
            raise RingDesyncError("IpcTransport.rx before reserve()")
        base = self.mail + (self.e & 1) * self.slot_bytes + self._off(tag)
        out, off = [], 0
        for t in likes:
            nb = t.numel() * t.element_size()
            if off + nb > self.caps[tag]:
                raise RingDesyncError(f"rank {self.rank}: receive of {off + nb} B exceeds the "
                                      f"reserved tag-{tag} region ({self.caps[tag]} B)")
            raw = torch.as_tensor(_DevBuf(base + off, nb), device=self.device)
            out.append(raw.view(t.dtype).view(t.shape))
            off += nb
        return out

    # ---------------------------------------------------------------- exchange
    def sendrecv(self, ops, stream):
        """Post one exchange (burst_ipc_ring_exchange: one C call, no host wait)."""
        import time
        t0 = time.perf_counter()
        if len(ops) > len(self._arr):
            self._arr = (_lib.IpcOp * (2 * len(ops)))()
        arr = self._arr
        for i, op in enumerate(ops):
            t = op[1]
            a = arr[i]
            a.buf = t.data_ptr()
            a.bytes = t.numel() * t.element_size()
            a.peer = op[2]
            a.is_send = 1 if op[0] == SEND else 0
            a.tag = op[3] if len(op) > 3 else TAG_ROT
        self.e += 1
        t1 = time.perf_counter()
        _lib.check(self._exchange(self.ring, arr, len(ops), ctypes.c_void_p(stream.cuda_stream)))
        self.c_us.append((time.perf_counter() - t1) * 1e6)
        ev = self._events[self.e & 1]
        ev.record(stream)
        self.last_wait = ev
        self.host_us.append((time.perf_counter() - t0) * 1e6)

    def finish(self, check: str) -> None:
        """"sync": wait (bounded) for the newest exchange; a peer that never signals
        leaves the comm stream blocked, reported as DeadlockError (sim.py:290-310)."""
        if check != "sync" or self.last_wait is None:
            return
        import time
        deadline = time.monotonic() + self.timeout_s
        while not self.last_wait.query():
            if time.monotonic() > deadline:
                raise DeadlockError(f"rank {self.rank}: IPC ring exchange {self.e - 1} did not "
                                    f"complete within {self.timeout_s:.0f} s")
            time.sleep(1e-4)

    def close(self):
        lib = _lib.load()
        torch.cuda.synchronize(self.device)
        for ptr in list(self.peer_mail.values()) + list(self.peer_flags.values()):
            lib.burst_ipc_close_mem(ctypes.c_void_p(ptr))
        self.peer_mail, self.peer_flags = {}, {}
        self.dist.barrier(group=self.group)     # every peer unmapped before freeing
        mine = [self.mail] if self.mail is not None else []
        for ptr in mine + self.retired + [self.flags, self.stage]:
            lib.burst_ipc_free(ctypes.c_void_p(ptr))
        self.mail, self.retired = None, []
        if self.ring:
            lib.burst_ipc_ring_destroy(self.ring)
            self.ring = None


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
               for kind, t, peer, *_ in ops]
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
            for kind, t, peer, *_ in ops:
                if kind == SEND:
                    ev = None
                    if cuda:
                        ev = torch.cuda.Event()
                        ev.record(stream)
                    hub.box[(seq, self.rank, peer)].append((t, ev))
        self._sync()
        taken = defaultdict(int)
        for kind, t, peer, *_ in ops:
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
        return [(SEND, self.send[i], (self.r + 1) % self.G, TAG_HDR),
                (RECV, self.log[i], (self.r - 1) % self.G, TAG_HDR)]

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


def _nbytes(*ts) -> int:
    return sum(t.numel() * t.element_size() for t in ts)


def _recv_bufs(transport, likes, tag: int, spare, device=None):
    """Receive targets of the next exchange: views of the transport's mailbox slot
    (mailbox transports receive in place) or the engine's own buffers (`spare`,
    allocated on first use and recycled by the caller).  `likes` give shape and
    dtype (meta tensors allowed, with `device` naming where to allocate)."""
    if transport.mailbox:
        return list(transport.rx(likes, tag))
    if spare is None:
        spare = [torch.empty(t.shape, dtype=t.dtype, device=device if device is not None else t.device)
                 for t in likes]
    return list(spare)


def _rotating(G: int, offset: int = 0):
    """origin_fn of a pass whose payload rotates at slots h < G-1 (K/V, or Q/dO); slot
    SHIFT (start offset) carries the sender's own block."""
    return lambda rank, h: (rank if h == SHIFT else
                            (rank - offset - h) % G if h < G - 1 else -1)


def backward_slots(G: int, offset: int = 0) -> list:
    """Exchange slots of a backward pass: the start-offset shift (SHIFT, only with an
    offset), K/V rotation at h < G-1, contribution homecoming (one hop late) at h >= 2,
    and the final homecoming slot G."""
    return (([SHIFT] if offset and G > 1 else []) +
            [h for h in range(G) if h < G - 1 or h >= _first_homecoming(offset)] +
            ([G] if G > 1 else []))


def _first_homecoming(offset: int) -> int:
    """Slot of the first contribution homecoming: hop h's contribution goes home at
    slot h + 1, except the own block's (hop 0 without a start offset)."""
    return 1 if offset else 2


SHIFT = -1      # exchange slot of the start-offset shift (before hop 0)


def _shift(transport, S, payload, tag: int, offset: int, slog, recorder, kind: str):
    """Start offset (initial_forward_body, ring.py:137-143; sim._initial_envelopes,
    sim.py:406-419): before hop 0 rank r sends its own rotating payload to r + offset
    and receives that of r - offset, so at hop h it holds block (r - offset - h) mod G.
    Returns the received payload (engine- or transport-owned buffers)."""
    G, r = transport.world, transport.rank
    got = _recv_bufs(transport, payload, tag, None)
    ops = ([(SEND, t, (r + offset) % G, tag) for t in payload] +
           [(RECV, t, (r - offset) % G, tag) for t in got])
    S.comm_after_compute()
    if recorder is not None:
        recorder.count_send(kind, ops)
    transport.sendrecv(ops + slog.ops(SHIFT), S.comm)
    S.compute_after_comm()
    return got


def ring_forward(q, k, v, scale: float, causal: bool, zigzag: bool, transport, kernels,
                 n_valid: int | None = None, recorder=None, grid=None, check: str = "sync",
                 offset: int = 0):
    """One rank's forward pass.  Returns (O [B,n,H,D], lse [B,H,n] natural log).
    `n_valid`: real global length when the shards are zero-padded (reference pad=True).
    `recorder`: optional trace.PassRecorder (measured timeline + ledger, sim.py:118-261).
    `grid`: optional masks.GridMask bound to the global length (BlockGrid).
    `check`: when the pass's device error word is read ("sync" | "async" | "off",
    kernels.finish; MaskError / NonFiniteError as in PartialAttn.finalize).
    `offset`: start offset (run_ring_pass(start_offset=...), sim.py:501-510): the merge
    order rotates, values agree to rounding."""
    B, n, H, D = q.shape
    G, r = transport.world, transport.rank
    offset %= G
    S = _Streams(q.device)
    o = torch.empty_like(q)
    lse = torch.empty(B, H, n, dtype=torch.float32, device=q.device)
    state = kernels.fwd_state(q, running=G > 1)
    slog = SlotLog(transport, q.device, ([SHIFT] if offset else []) + list(range(G - 1)),
                   _rotating(G, offset))
    if G > 1:
        transport.reserve({TAG_ROT: _nbytes(k, v), TAG_HDR: HDR_BYTES})
    cur_k, cur_v = k, v
    if offset:
        cur_k, cur_v = _shift(transport, S, (k, v), TAG_ROT, offset, slog, recorder, "forward")
    spare = None
    finalized = False
    computed = False             # a hop has merged into the running state
    prev = S.compute_mark()      # compute tail before hop h (buffers it still reads)
    for h in range(G):
        plan = plan_hop(r, G, h, n, causal, zigzag, n_valid, grid, offset)
        exchanged = False
        # launch the hop's kernel first, then post the transfer on the comm stream:
        # both run concurrently (the comm waits only for the PREVIOUS hop's kernel,
        # which last read the buffer being received into)
        if recorder is not None:
            recorder.mark(h, "compute_start", S.compute)
        if not plan.skip:
            fin = h == G - 1 and plan.covers_all_queries(n)
            first = not computed
            if first and not plan.covers_all_queries(n):
                # the rows this rectangle leaves out need a defined (empty) state
                kernels.fwd_init(state, stream=S.compute)
                first = False
            kernels.fwd(plan, q, cur_k, cur_v, scale, state, o, lse, first=first,
                        finalize=fin, stream=S.compute)
            finalized = finalized or fin
            computed = True
        if recorder is not None:
            recorder.mark(h, "compute_end", S.compute)
        done = S.compute_mark()
        if h < G - 1:
            spare = _recv_bufs(transport, (k, v), TAG_ROT, spare)
            S.comm_wait(prev)
            ops = [(SEND, cur_k, (r + 1) % G, TAG_ROT), (SEND, cur_v, (r + 1) % G, TAG_ROT),
                   (RECV, spare[0], (r - 1) % G, TAG_ROT), (RECV, spare[1], (r - 1) % G, TAG_ROT)]
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
                   recv_bufs, n_valid=None, grid=None, offset: int = 0):
    """Ops moving the dK/dV contribution computed at `hop` to its home rank, and
    receiving into `recv_bufs` the one computed for ours (none when the hop's block is
    the own block, which accumulates in place).  Returns (ops, received?)."""
    ops = []
    mine = plan_hop(r, G, hop, n, causal, zigzag, n_valid, grid, offset)
    if not mine.skip and mine.src != r:
        ops += [(SEND, send_bufs[0], mine.src, TAG_PART), (SEND, send_bufs[1], mine.src, TAG_PART)]
    c = contributor_to(r, G, hop, offset)
    got = c != r and not plan_hop(c, G, hop, n, causal, zigzag, n_valid, grid, offset).skip
    if got:
        ops += [(RECV, recv_bufs[0], c, TAG_PART), (RECV, recv_bufs[1], c, TAG_PART)]
    return ops, got


def ring_backward(q, k, v, o, lse, dout, scale: float, causal: bool, zigzag: bool, transport,
                  kernels, n_valid: int | None = None, recorder=None, grid=None,
                  check: str = "sync", deterministic: bool = False, offset: int = 0):
    """One rank's backward pass.  Returns (dq, dk, dv) in q's dtype.

    Contribution buffers are O(1) in the ring size: `own` accumulates this rank's
    dK/dV, `send[2]` hold the contributions of the last two hops (each goes home one
    hop later), `recv` the contribution arriving for our block, folded into `own`
    (burst_tl_accumulate) before the next hop -- the in-place accumulation of
    ring.backward_step (ring.py:239-241).  The own block is computed in two query
    halves (split_own_hop) so the final homecoming exchange overlaps a kernel.
    `recorder`: optional trace.PassRecorder (see ring_forward).  `offset`: start
    offset (K/V start shifted, see ring_forward); the own block then comes at hop
    G - offset and is not split."""
    B, n, H, D = q.shape
    G, r = transport.world, transport.rank
    offset %= G
    S = _Streams(q.device)
    st = kernels.bwd_prepare(o, dout, lse, stream=S.compute, deterministic=deterministic)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    own = (kernels.part(k), kernels.part(v))
    slog = SlotLog(transport, q.device, backward_slots(G, offset), _rotating(G, offset))
    if G > 1:
        transport.reserve({TAG_ROT: _nbytes(k, v), TAG_PART: _nbytes(*own), TAG_HDR: HDR_BYTES})
    send = [None, None]
    recv = None                  # contribution receive buffers (engine-owned or mailbox views)
    pending = False              # `recv` holds a contribution not yet folded into `own`
    own_last = None              # second query half of the own block (after hop G-1)
    own_ready = False            # `own` holds a defined value
    cur_k, cur_v = k, v
    if offset:
        cur_k, cur_v = _shift(transport, S, (k, v), TAG_ROT, offset, slog, recorder, "backward")
    spare = None

    def fold():
        nonlocal own_ready
        if own_ready:
            kernels.accumulate(own, recv, k, stream=S.compute)
        else:                    # (offset) a contribution landed before the own block ran
            with torch.cuda.stream(S.compute) if S.cuda else _nullctx():
                own[0].copy_(recv[0])
                own[1].copy_(recv[1])
            own_ready = True

    for h in range(G):
        plan = plan_hop(r, G, h, n, causal, zigzag, n_valid, grid, offset)
        if h == 0 and not offset:
            plan, own_last = split_own_hop(plan, n, G)
        if recorder is not None:
            recorder.mark(h, "compute_start", S.compute)
        if pending:              # landed in the previous slot (compute waited for it)
            fold()
            pending = False
        # this slot's transfers wait for everything above: hop h-1's kernel (it made
        # the contribution sent now and last read `spare`) and the fold of `recv`
        ready = S.compute_mark()
        is_own = plan.src == r
        if is_own:
            target = own
        else:
            if send[h % 2] is None:
                send[h % 2] = (kernels.part(k), kernels.part(v))
            target = send[h % 2]
        if not plan.skip:
            kernels.bwd(plan, q, cur_k, cur_v, dout, scale, st, target[0], target[1],
                        accumulate=is_own and own_ready, stream=S.compute)
            own_ready = own_ready or is_own
        elif is_own and not own_ready:   # own block fully masked (grid): no contribution
            kernels.zero_(target, stream=S.compute)
            own_ready = True
        if recorder is not None:
            recorder.mark(h, "compute_end", S.compute)
        ops = []
        if h < G - 1:
            spare = _recv_bufs(transport, (k, v), TAG_ROT, spare)
            ops += [(SEND, cur_k, (r + 1) % G, TAG_ROT), (SEND, cur_v, (r + 1) % G, TAG_ROT),
                    (RECV, spare[0], (r - 1) % G, TAG_ROT), (RECV, spare[1], (r - 1) % G, TAG_ROT)]
        if h >= _first_homecoming(offset):
            recv = _recv_bufs(transport, own, TAG_PART, recv)
            p_ops, got = _part_exchange(r, G, n, causal, zigzag, h - 1, send[(h - 1) % 2],
                                        recv, n_valid, grid, offset)
            ops += p_ops
            pending = got
        # every rank takes part in every exchange slot (a slot depends only on
        # h and G), even with no op of its own: keeps loopback/collective
        # transports in lockstep when causal hops are skipped
        slot = h < G - 1 or h >= _first_homecoming(offset)
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
            fold()
        ready = S.compute_mark()
        recv = _recv_bufs(transport, own, TAG_PART, recv)
        p_ops, got = _part_exchange(r, G, n, causal, zigzag, G - 1, send[(G - 1) % 2], recv,
                                    n_valid, grid, offset)
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
                    recv_buf, n_valid=None, grid=None, offset: int = 0):
    """Ops moving the dQ contribution computed at `hop` (for the visiting query
    block) to that block's home rank, and receiving into `recv_buf` the one
    computed for ours (none for the own block).  Returns (ops, received?)."""
    ops = []
    src = (r - offset - hop) % G               # origin of the query block I processed
    if src != r and not plan_hop(src, G, (src - r) % G, n, causal, zigzag, n_valid, grid).skip:
        ops.append((SEND, send_buf, src, TAG_PART))
    c = (r + offset + hop) % G                 # the rank that processed MY block at `hop`
    got = c != r and not plan_hop(r, G, (r - c) % G, n, causal, zigzag, n_valid, grid).skip
    if got:
        ops.append((RECV, recv_buf, c, TAG_PART))
    return ops, got


def ring_backward_qtravel(q, k, v, o, lse, dout, scale: float, causal: bool, zigzag: bool,
                          transport, kernels, n_valid: int | None = None, recorder=None,
                          grid=None, check: str = "sync", deterministic: bool = False,
                          offset: int = 0):
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
    fp32 dK/dV for ring_backward.  `offset`: start offset (the query record of rank
    r - offset starts on rank r, sim._initial_envelopes sim.py:406-419).  Returns
    (dq, dk, dv) in q's dtype."""
    B, n, H, D = q.shape
    G, r = transport.world, transport.rank
    offset %= G
    S = _Streams(q.device)
    st = kernels.bwd_prepare(o, dout, lse, stream=S.compute, deterministic=deterministic)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    dk_acc, dv_acc = kernels.part(k), kernels.part(v)
    payload = [q, dout] + kernels.stats_tensors(st)      # the visiting query block
    slog = SlotLog(transport, q.device, backward_slots(G, offset), _rotating(G, offset))
    if G > 1:
        dq_like = kernels.dq_like(q)         # shape/dtype of a dQ contribution (meta)
        transport.reserve({TAG_ROT: _nbytes(*payload), TAG_PART: _nbytes(dq_like),
                           TAG_HDR: HDR_BYTES})
    if offset:
        payload = _shift(transport, S, payload, TAG_ROT, offset, slog, recorder, "backward")
    spare = None
    send = [None, None]
    recv = None                  # dQ contribution receive buffer (engine-owned or a mailbox view)
    pending = False
    own_last = None
    first_kv = True
    for h in range(G):
        src = (r - offset - h) % G
        plan = plan_hop(src, G, (src - r) % G, n, causal, zigzag, n_valid, grid)
        if h == 0 and not offset:
            plan, own_last = split_own_hop(plan, n, G)
        if recorder is not None:
            recorder.mark(h, "compute_start", S.compute)
        if pending:
            kernels.accumulate_dq(st, recv, q, stream=S.compute)
            pending = False
        ready = S.compute_mark()
        if src == r:
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
            spare = _recv_bufs(transport, payload, TAG_ROT, spare)
            ops += [(SEND, t, (r + 1) % G, TAG_ROT) for t in payload]
            ops += [(RECV, t, (r - 1) % G, TAG_ROT) for t in spare]
        if h >= _first_homecoming(offset):
            recv = _recv_bufs(transport, (dq_like,), TAG_PART,
                              None if recv is None else (recv,), q.device)[0]
            p_ops, got = _qpart_exchange(r, G, n, causal, zigzag, h - 1, send[(h - 1) % 2],
                                         recv, n_valid, grid, offset)
            ops += p_ops
            pending = got
        slot = h < G - 1 or h >= _first_homecoming(offset)
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
        recv = _recv_bufs(transport, (dq_like,), TAG_PART,
                          None if recv is None else (recv,), q.device)[0]
        p_ops, got = _qpart_exchange(r, G, n, causal, zigzag, G - 1, send[(G - 1) % 2], recv,
                                     n_valid, grid, offset)
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
