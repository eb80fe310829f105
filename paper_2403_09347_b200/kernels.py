"""Kernel provider: torch tensors in, C-ABI (libburst_b200.so) calls out.

This is the ONLY compute provider of the product.  Every method checks that
its tensors live on a CUDA device and raises otherwise: there is no CPU path.
The ring engine (`ring.py`) sees the running forward state and backward
workspaces as opaque objects created here.

Mapping onto the reference (pkg/src/burstsim):
  fwd           ring.forward_step -> local_forward_tiled + PartialAttn.merge
  fwd_finalize  PartialAttn.finalize / ring.finalize_forward
  bwd_prepare   ring.init_backward (D = rowsum(dO * O), zeroed dQ accumulator)
  bwd           ring.backward_step -> local_backward
  bwd_finalize  sim._collect (dQ home, dK/dV summed)
"""

from __future__ import annotations

import ctypes
import math
import threading
from dataclasses import dataclass

import torch

from . import _lib
from .errors import CudaError, MaskError, NonFiniteError, ShapeError
from .schedule import HopPlan

_DTYPES = {torch.bfloat16: _lib.DTYPE_BF16, torch.float32: _lib.DTYPE_F32}


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream_handle(stream) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _DTYPES[t.dtype]
    except KeyError:
        raise ShapeError(f"unsupported dtype {t.dtype}; use bfloat16 or float32") from None


def check_qkv(q, k, v) -> tuple[int, int, int, int]:
    """[B, n, H, D] contiguous CUDA tensors of one dtype (dense.py:34-46 checks)."""
    for name, t in (("q", q), ("k", k), ("v", v)):
        if not t.is_cuda:
            raise CudaError(f"{name} is on {t.device}: the BurstAttention path runs only on CUDA "
                            "(sm_100a); there is no CPU fallback")
        if t.dim() != 4:
            raise ShapeError(f"{name} must be [batch, seq, heads, head_dim], got {tuple(t.shape)}")
        if not t.is_contiguous():
            raise ShapeError(f"{name} must be contiguous")
    if q.dtype != k.dtype or q.dtype != v.dtype:
        raise ShapeError("mixed dtypes across Q, K, V")
    if k.shape != v.shape or q.shape[0] != k.shape[0] or q.shape[2:] != k.shape[2:]:
        raise ShapeError(f"incompatible shapes Q={tuple(q.shape)} K={tuple(k.shape)} "
                         f"V={tuple(v.shape)}")
    B, n, H, D = q.shape
    if n < 1 or k.shape[1] < 1:
        raise ShapeError("empty attention block")
    dtype_code(q)
    return B, n, H, D




def ws_floats(B: int, H: int, D: int, n: int) -> int:
    return B * H * (-(-n // 128) * 128) * D


@dataclass
class FwdState:
    """Running (O_acc, m, l) of the pinned query block (PartialAttn, local_attn.py:66-99),
    None for a one-hop pass, and the pass's device error word."""
    o_acc: torch.Tensor | None   # TL fp32 workspace
    m: torch.Tensor | None       # [B, H, n] fp32, log2 units
    l: torch.Tensor | None       # [B, H, n] fp32
    flags: torch.Tensor          # [1] int32 (burst_hop.flags)


@dataclass
class BwdState:
    stats: torch.Tensor   # flat [2][B*H][ceil(n/128)*128] (lse*log2e, D)
    dq_acc: torch.Tensor  # TL fp32
    flags: torch.Tensor   # [1] int32 error word of the pass
    order: torch.Tensor | None = None   # deterministic mode: burst_hop.dq_order (selector)


# bits of the device error word (include/burst_b200.h burst_hop.flags)
FLAG_MASK, FLAG_NONFINITE, FLAG_LAUNCH = 1, 2, 4


def raise_for_flags(bits: int, where: str) -> None:
    """Map the device error word onto the reference taxonomy: MaskError first (a row
    with no visible key), then NonFiniteError (PartialAttn.finalize order,
    local_attn.py:127-135; linalg._ensure_finite, linalg.py:253-255)."""
    if bits & FLAG_MASK:
        raise MaskError(f"{where}: some query row accumulated no unmasked entries")
    if bits & FLAG_NONFINITE:
        raise NonFiniteError(f"{where} produced a non-finite value")
    if bits & FLAG_LAUNCH:
        raise CudaError(f"{where}: a kernel could not run (shared-memory alignment)")


class _Pending:
    """Error words copied to pinned host memory at the end of passes run with
    check="async"; raised at the next pass entry once the copy has landed, or by
    check_errors() (blocking)."""

    def __init__(self):
        self.lock = threading.Lock()
        self.items = []      # (host tensor, event, checker(host) -> raises)

    def add(self, flags: torch.Tensor, stream, where: str) -> None:
        self.add_check(flags, stream, lambda h: raise_for_flags(int(h[0]), where))

    def add_check(self, dev: torch.Tensor, stream, checker) -> None:
        """Copy `dev` to pinned host memory on `stream`; run checker(host) once it lands."""
        host = torch.empty(dev.shape, dtype=dev.dtype, pin_memory=True)
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            host.copy_(dev, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
        with self.lock:
            self.items.append((host, ev, checker))

    def check(self, block: bool) -> None:
        with self.lock:
            items, keep, ready = self.items, [], []
            for host, ev, checker in items:
                if block:
                    ev.synchronize()
                elif not ev.query():
                    keep.append((host, ev, checker))
                    continue
                ready.append((host, checker))
            self.items = keep
        for host, checker in ready:   # raises the first error; the rest are dropped
            checker(host)


PENDING = _Pending()


def check_errors() -> None:
    """Raise the first error recorded by an asynchronously checked pass (blocks until
    every such pass has finished on the device)."""
    PENDING.check(block=True)


def make_hop(plan: HopPlan, q: torch.Tensor, k: torch.Tensor, scale: float,
             flags: torch.Tensor | None = None, order: torch.Tensor | None = None) -> _lib.Hop:
    B, n_q, H, D = q.shape
    h = _lib.Hop()
    h.batch, h.heads, h.head_dim, h.dtype = B, H, D, dtype_code(q)
    h.n_q, h.n_k = n_q, k.shape[1]
    h.q_begin, h.q_len, h.k_begin, h.k_len = plan.q_begin, plan.q_len, plan.k_begin, plan.k_len
    h.softmax_scale = float(scale)
    h.causal = 1 if plan.causal else 0
    h.q_map = _lib.PosMap(plan.q_map.pos0, plan.q_map.pos1, plan.q_map.seg_len)
    h.k_map = _lib.PosMap(plan.k_map.pos0, plan.k_map.pos1, plan.k_map.seg_len)
    g = plan.grid
    if g is not None:
        # keeps the table alive: GridMask.device_table caches it per device
        h.grid_skip = g.device_table(q.device).data_ptr()
        h.grid_nqb, h.grid_nkb = g.n_query_blocks, g.n_key_blocks
        h.grid_qcell, h.grid_kcell = g.qcell, g.kcell
    if flags is not None:
        h.flags = flags.data_ptr()
    if order is not None:
        h.dq_order = order.data_ptr()
    if plan.key_order is not None:
        h.key_order = plan.key_order.data_ptr()
    return h


class CudaKernels:
    """sm_100a kernels behind the C ABI (tcgen05 bf16 / SIMT f32)."""

    name = "cuda"

    def __init__(self):
        _lib.load()

    # ------------------------------------------------------------ allocation
    @staticmethod
    def _flags(device) -> torch.Tensor:
        return torch.zeros(1, dtype=torch.int32, device=device)

    def fwd_state(self, q: torch.Tensor, running: bool = True) -> FwdState:
        """Running state of a pass (none needed when one hop finalizes directly)."""
        B, n, H, D = q.shape
        dev = q.device
        if not running:
            return FwdState(None, None, None, self._flags(dev))
        return FwdState(torch.empty(ws_floats(B, H, D, n), dtype=torch.float32, device=dev),
                        torch.empty(B, H, n, dtype=torch.float32, device=dev),
                        torch.empty(B, H, n, dtype=torch.float32, device=dev),
                        self._flags(dev))

    def part(self, k: torch.Tensor) -> torch.Tensor:
        """One fp32 dK or dV contribution buffer for a visiting block (TL layout)."""
        B, n, H, D = k.shape
        return torch.empty(ws_floats(B, H, D, n), dtype=torch.float32, device=k.device)

    # ------------------------------------------------------------ forward
    def fwd(self, plan: HopPlan, q, k, v, scale: float, state: FwdState | None, o, lse,
            first: bool, finalize: bool, stream=None) -> None:
        """One hop; `state` None: a single finalizing hop on the per-device error word."""
        st = state if state is not None else FwdState(None, None, None, None)
        hop = make_hop(plan, q, k, scale, st.flags)
        _lib.call("burst_lao_fwd", ctypes.byref(hop), _ptr(q), _ptr(k), _ptr(v),
                  _ptr(st.o_acc), _ptr(st.m), _ptr(st.l), _ptr(o if finalize else None),
                  _ptr(lse if finalize else None), int(first), int(finalize),
                  _stream_handle(stream))

    def fwd_init(self, state: FwdState, stream=None) -> None:
        """Empty running state (PartialAttn.empty, local_attn.py:66-99): O_acc = 0,
        m = -inf, l = 0, for a pass whose first computed hop covers only part of the
        query block (start offset or a masked own block: Q_LATE_HALF comes first)."""
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            state.o_acc.zero_()
            state.m.fill_(float("-inf"))
            state.l.zero_()

    def fwd_finalize(self, state: FwdState, o, lse, stream=None) -> None:
        B, n, H, D = o.shape
        _lib.call("burst_fwd_finalize", dtype_code(o), B, H, D, n, _ptr(state.o_acc),
                  _ptr(state.m), _ptr(state.l), _ptr(o), _ptr(lse), _ptr(state.flags),
                  _stream_handle(stream))

    # ------------------------------------------------------------ error boundary
    def finish(self, state, check: str, stream=None, where: str = "BurstAttention") -> None:
        """Read the pass's device error word once: "sync" raises here (synchronises
        the stream), "async" copies it to pinned memory and raises at a later pass
        entry or in check_errors(), "off" skips the check."""
        if check == "off":
            return
        if check == "sync":
            s = stream if stream is not None else torch.cuda.current_stream()
            s.synchronize()
            raise_for_flags(int(state.flags.item()), where)
        elif check == "async":
            PENDING.add(state.flags, stream, where)
        else:
            raise ValueError(f"check must be 'sync', 'async' or 'off', got {check!r}")

    # ------------------------------------------------------------ backward
    def bwd_prepare(self, o, dout, lse, stream=None, deterministic: bool = False) -> BwdState:
        """Backward stats + zeroed dQ accumulator of the pinned block; `deterministic`
        also selects the bit-reproducible backward (dK/dV key-stationary, dQ query-stationary)."""
        B, n, H, D = o.shape
        nt = -(-n // 128) * 128
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            flags = self._flags(o.device)
        # [2][B*H][nt]: the backward loads whole 128-row tiles of the block (padded rows
        # are written by burst_bwd_preprocess), never past the last tile
        stats = torch.empty(2 * B * H * nt, dtype=torch.float32, device=o.device)
        order = (torch.empty(B * H * (-(-n // 128)), dtype=torch.int32, device=o.device)
                 if deterministic else None)
        st = BwdState(stats,
                      torch.empty(ws_floats(B, H, D, n), dtype=torch.float32, device=o.device),
                      flags, order)
        _lib.call("burst_bwd_preprocess", dtype_code(o), B, H, D, n, _ptr(o), _ptr(dout),
                  _ptr(lse), _ptr(st.stats), _ptr(st.dq_acc), _stream_handle(stream))
        return st

    def bwd(self, plan: HopPlan, q, k, v, dout, scale: float, st: BwdState, dk_part, dv_part,
            accumulate: bool, stream=None) -> None:
        hop = make_hop(plan, q, k, scale, st.flags, st.order)
        _lib.call("burst_lao_bwd", ctypes.byref(hop), _ptr(q), _ptr(k), _ptr(v), _ptr(dout),
                  _ptr(st.stats), _ptr(st.dq_acc), _ptr(dk_part), _ptr(dv_part), int(accumulate),
                  _stream_handle(stream))

    def accumulate(self, acc_pair, part_pair, like: torch.Tensor, stream=None) -> None:
        """acc += part for a (dK, dV) pair of TL contribution buffers."""
        B, n, H, D = like.shape
        for a, p in zip(acc_pair, part_pair):
            _lib.call("burst_tl_accumulate", B, H, D, n, _ptr(a), _ptr(p), _stream_handle(stream))

    def bwd_finalize(self, st: BwdState, dk_parts, dv_parts, dq, dk, dv, stream=None) -> None:
        B, n, H, D = dq.shape
        np_ = len(dk_parts)
        arr_k = (ctypes.c_void_p * max(np_, 1))(*[p.data_ptr() for p in dk_parts])
        arr_v = (ctypes.c_void_p * max(np_, 1))(*[p.data_ptr() for p in dv_parts])
        _lib.call("burst_bwd_finalize", dtype_code(dq), B, H, D, n, _ptr(st.dq_acc), arr_k, arr_v,
                  np_, _ptr(dq), _ptr(dk), _ptr(dv), _ptr(st.flags), _stream_handle(stream))

    # ------------------------------------------------ travelling-query backward (f2)
    def stats_tensors(self, st: BwdState) -> list:
        """The per-query-block backward statistics that travel with Q and dO."""
        return [st.stats]

    def visiting_state(self, st: BwdState, stats: list, dq_part) -> BwdState:
        """Backward state of a visiting query block: its statistics, and the fresh
        dQ contribution buffer this hop reduces into."""
        return BwdState(stats[0], dq_part, st.flags, st.order)

    def dq_part(self, q: torch.Tensor, stream=None, reuse: torch.Tensor | None = None) -> torch.Tensor:
        """A zeroed fp32 dQ contribution buffer (TL layout) for a visiting block,
        zeroed on `stream` (`reuse`: an earlier buffer to zero again)."""
        B, n, H, D = q.shape
        buf = reuse if reuse is not None else torch.empty(ws_floats(B, H, D, n),
                                                          dtype=torch.float32, device=q.device)
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            buf.zero_()
        return buf

    def dq_like(self, q: torch.Tensor) -> torch.Tensor:
        """Shape/dtype of a dQ contribution buffer (a meta tensor: no memory)."""
        B, n, H, D = q.shape
        return torch.empty(ws_floats(B, H, D, n), dtype=torch.float32, device="meta")

    def accumulate_dq(self, st: BwdState, part: torch.Tensor, like: torch.Tensor,
                      stream=None) -> None:
        """Fold a received dQ contribution into the home dQ accumulator."""
        B, n, H, D = like.shape
        _lib.call("burst_tl_accumulate", B, H, D, n, _ptr(st.dq_acc), _ptr(part),
                  _stream_handle(stream))

    def tl_sum(self, parts, out, flags=None, stream=None) -> None:
        B, n, H, D = out.shape
        arr = (ctypes.c_void_p * len(parts))(*[p.data_ptr() for p in parts])
        _lib.call("burst_tl_sum", dtype_code(out), B, H, D, n, arr, len(parts), _ptr(out),
                  _ptr(flags), _stream_handle(stream))

    def bwd_finalize_qtravel(self, st: BwdState, dq_parts, dk_acc, dv_acc, dq, dk, dv,
                             stream=None) -> None:
        """dq = own accumulator + received contributions; dk/dv = pinned accumulators."""
        self.tl_sum([st.dq_acc] + list(dq_parts), dq, st.flags, stream)
        self.tl_sum([dk_acc], dk, st.flags, stream)
        self.tl_sum([dv_acc], dv, st.flags, stream)

    def zero_(self, bufs, stream=None) -> None:
        """Zero contribution buffers on `stream` (a fully masked own block)."""
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            for b in bufs:
                b.zero_()



def default_scale(head_dim: int) -> float:
    """softmax scale d^-0.5 (runner.py:154)."""
    return 1.0 / math.sqrt(head_dim)


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
