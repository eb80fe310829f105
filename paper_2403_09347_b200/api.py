"""Public entry points.

`burst_attn_func(q, k, v, causal, softmax_scale, group)` is the drop-in
attention call of the north star: q/k/v are this rank's sequence shards
[batch, n_local, heads, head_dim]; it returns (out, lse) and is differentiable
(autograd backward = the ring backward).  It replaces the reference's pass-level
run_ring_pass forward+backward (sim.py:501-657) for one rank.

`run_ring_pass` / `burst_attn_global` run a whole G-device ring inside one
process on one GPU (loopback transport, one thread per simulated device) and
mirror the reference's pass-level API for parity tests.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .errors import ConfigError, ShapeError
from .masks import GridMask
from .kernels import PENDING, CudaKernels, check_errors, check_qkv, default_scale
from .ring import (IpcTransport, NcclTransport, SoloTransport, ring_backward,
                   ring_backward_qtravel, ring_forward, run_ranks)
from .schedule import shard, unshard
from .trace import PassRecorder, PassTrace, merge

_kernels = None
_transports = {}


def _default_kernels():
    global _kernels
    if _kernels is None:
        _kernels = CudaKernels()
    return _kernels


def _transport_for(group, comm: str = "nccl", deadlock_timeout: float | None = None):
    """Ring transport of `group`: "nccl" (NCCL send/recv kernels) or "ce" (zero-SM
    copy-engine pushes into CUDA-IPC mailboxes, ring.IpcTransport)."""
    import torch.distributed as dist
    if group is None and not (dist.is_available() and dist.is_initialized()):
        return SoloTransport()
    world = dist.get_world_size(group)
    if world == 1:
        return SoloTransport()
    if comm not in ("nccl", "ce"):
        raise ConfigError(f"comm must be 'nccl' or 'ce', got {comm!r}")
    key = (id(group), torch.cuda.current_device(), comm, deadlock_timeout)
    if key not in _transports:
        _transports[key] = (NcclTransport(group, timeout_s=deadlock_timeout) if comm == "nccl"
                            else IpcTransport(group, timeout_s=deadlock_timeout))
    return _transports[key]


class _BurstAttnFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, scale, causal, zigzag, transport, kernels, n_valid, recorders,
                bwd_payload, grid, check, deterministic, offset):
        rec_f, rec_b = recorders if recorders is not None else (None, None)
        o, lse = ring_forward(q, k, v, scale, causal, zigzag, transport, kernels, n_valid,
                              recorder=rec_f, grid=grid, check=check, offset=offset)
        ctx.save_for_backward(q, k, v, o, lse)
        ctx.cfg = (scale, causal, zigzag, transport, kernels, n_valid, rec_b, bwd_payload, grid,
                   check, deterministic, offset)
        ctx.mark_non_differentiable(lse)
        ctx.set_materialize_grads(False)     # no zero dlse tensor per backward
        return o, lse

    @staticmethod
    def backward(ctx, do, _dlse):
        q, k, v, o, lse = ctx.saved_tensors
        (scale, causal, zigzag, transport, kernels, n_valid, rec_b, bwd_payload, grid, check,
         deterministic, offset) = ctx.cfg
        if do is None:
            return (None,) * 15
        bwd = ring_backward_qtravel if bwd_payload == "q" else ring_backward
        dq, dk, dv = bwd(q, k, v, o, lse, do.contiguous(), scale, causal, zigzag, transport,
                         kernels, n_valid, recorder=rec_b, grid=grid, check=check,
                         deterministic=deterministic, offset=offset)
        return (dq, dk, dv) + (None,) * 12


def burst_attn_func(q, k, v, causal: bool = False, softmax_scale: float | None = None,
                    group=None, zigzag: bool | None = None, valid_len: int | None = None, *,
                    bwd_payload: str = "kv", mask=None, comm: str = "nccl", check: str = "async",
                    deadlock_timeout: float | None = None, deterministic: bool = False,
                    start_offset: int = 0, _transport=None, _kernels=None, _recorders=None):
    """BurstAttention over the ranks of `group` (NCCL ring over NVLink).

    q, k, v: [batch, n_local, heads, head_dim] shards of the global sequence
    (contiguous blocks, or zigzag chunks {rank, 2G-1-rank} when causal and
    zigzag -- the default for causal with G > 1; see `schedule.shard`).
    Returns (out [batch, n_local, heads, head_dim], lse [batch, heads, n_local]).
    `valid_len`: real global sequence length when the shards were zero-padded to
    a multiple of G (2G for zigzag); padded keys are excluded, padded rows of the
    outputs are meaningless (the reference's pad=True, ring.py:111-115).
    `bwd_payload`: "kv" (default) rotates K/V and sends fp32 dK/dV contributions
    home; "q" is the reference's payload (Q, dO, lse/D travel, K/V/dK/dV pinned,
    ring.py:65-83) with fp32 dQ contributions sent home.
    `mask`: block-sparse grid over the GLOBAL score matrix -- a masks.GridMask or a
    mask_from_spec value (dict / JSON path with n_query_blocks, n_key_blocks, skip and
    an optional causal flag; masking.py:150-180); composes with `causal`.
    `comm`: ring transport, "nccl" (default) or "ce" (copy engines + CUDA IPC, no SM).
    `check`: when each pass's device error word (MaskError: a row with no visible key;
    NonFiniteError: a non-finite output) is read: "async" (default) raises at a later
    call once the pass has finished on the device, or in `check_errors()`, without
    stalling the host; "sync" raises at the end of each pass (synchronises); "off".
    `deadlock_timeout`: seconds without any ring exchange completing before the NCCL
    communicator is aborted and the pass raises DeadlockError (default
    BURST_RING_TIMEOUT_S or 600; the reference's deadlock_timeout, sim.py:501-510).
    Every exchange also carries a small header checked at pass end (RingDesyncError).
    `deterministic`: dQ from a query-stationary kernel that sums each row over the key
    tiles in order (one writer per row) so gradients are bit-reproducible run to run
    and across transports (the reference's bitwise executor equivalence,
    pkg/tests/test_sim.py:280-295); ~1/3 slower backward.
    `start_offset`: rank r starts the ring with the K/V block of rank r - start_offset
    (mod G) instead of its own (initial_forward_body, ring.py:137-143); one extra
    exchange, the merge order rotates and values agree to rounding.
    `_recorders`: optional (forward, backward) trace.PassRecorder pair that
    records this rank's measured hop timeline and byte ledger.
    """
    PENDING.check(block=False)      # errors of earlier asynchronously checked passes
    check_qkv(q, k, v) if _kernels is None else None
    if q.shape[1] != k.shape[1]:
        raise ShapeError("ring shards must have equal query and key lengths")
    scale = default_scale(q.shape[-1]) if softmax_scale is None else float(softmax_scale)
    if not scale > 0:
        raise ShapeError(f"scale must be finite and positive, got {scale}")
    transport = (_transport if _transport is not None
                 else _transport_for(group, comm, deadlock_timeout))
    kernels = _kernels if _kernels is not None else _default_kernels()
    if zigzag is None:
        zigzag = bool(causal) and transport.world > 1
    if zigzag and q.shape[1] % 2:
        raise ShapeError("zigzag shards need an even local length")
    if zigzag and q.dtype == torch.bfloat16 and (q.shape[1] // 2) % 8:
        # the Q_LATE_HALF hop starts at the chunk boundary; the bf16 kernels need it
        # 8-row aligned.  Rejected here, on every rank, before any exchange is posted
        raise ShapeError(f"bf16 zigzag shards need a chunk length (n_local / 2 = "
                         f"{q.shape[1] // 2}) that is a multiple of 8")
    if check not in ("sync", "async", "off"):
        raise ConfigError(f"check must be 'sync', 'async' or 'off', got {check!r}")
    if valid_len is not None and not 0 < valid_len <= q.shape[1] * transport.world:
        raise ShapeError(f"valid_len={valid_len} outside (0, {q.shape[1] * transport.world}]")
    if bwd_payload not in ("kv", "q"):
        raise ConfigError(f"bwd_payload must be 'kv' or 'q', got {bwd_payload!r}")
    grid, causal = _bind_mask(mask, causal, q.shape[1] * transport.world, valid_len)
    return _BurstAttnFn.apply(q, k, v, scale, bool(causal), bool(zigzag), transport, kernels,
                              valid_len, _recorders, bwd_payload, grid, check,
                              bool(deterministic), _offset(start_offset))


def _offset(start_offset) -> int:
    """The reference takes any integer start offset modulo G (sim.py:414)."""
    if isinstance(start_offset, bool) or not isinstance(start_offset, int):
        raise ConfigError(f"start_offset must be an integer, got {start_offset!r}")
    return start_offset


def _bind_mask(mask, causal, total, n_valid=None):
    """(GridMask bound to the global (padded) length or None, effective causal flag);
    validates that every real query row keeps a visible key (BlockMask.validate,
    masking.py:132-147)."""
    if mask is None:
        return None, causal
    if isinstance(mask, GridMask):
        grid, spec_causal = mask, False
    else:
        grid, spec_causal = GridMask.from_spec(mask)
    causal = bool(causal) or spec_causal
    if grid is None:
        return None, causal
    grid = grid.bind(total)
    grid.validate(causal, n_valid)
    return grid, causal


@dataclass
class PassResult:
    """Mirror of sim.PassResult (sim.py:386-397): outputs and grads, global order."""
    out: torch.Tensor
    lse: torch.Tensor
    dq: torch.Tensor | None = None
    dk: torch.Tensor | None = None
    dv: torch.Tensor | None = None
    trace: object | None = None     # trace.PassTrace when run_ring_pass(trace=True)


def run_ring_pass(q, k, v, world: int, causal: bool = False, softmax_scale: float | None = None,
                  dout=None, zigzag: bool | None = None, kernels=None,
                  pad: bool = False, trace: bool = False,
                  bwd_payload: str = "kv", mask=None, check: str = "sync",
                  deadlock_timeout: float | None = None,
                  deterministic: bool = False, start_offset: int = 0) -> PassResult:
    """Whole-ring forward (+ backward when `dout` is given) of GLOBAL tensors
    [batch, N, heads, head_dim] over `world` simulated devices on this GPU.

    Mirrors build_cluster + run_ring_pass (sim.py:366-383, 501-657) with the
    threaded executor: one thread per device, real CUDA kernels, device
    copies for the ring hand-off.  `trace=True` also returns the measured
    per-hop timeline and byte ledger of every device (`.trace`, a
    trace.PassTrace in the reference's ScheduleTrace / CommLedger schema).
    `deadlock_timeout`: seconds a rank waits for its peers at an exchange before the
    pass raises DeadlockError (the reference's deadlock_timeout, sim.py:501-510).
    `deterministic`: bit-reproducible backward (see burst_attn_func).
    `start_offset`: rotated initial K/V assignment (see burst_attn_func).
    """
    if world < 1:
        raise ConfigError(f"gpus must be a positive integer, got {world}")
    if bwd_payload not in ("kv", "q"):
        raise ConfigError(f"bwd_payload must be 'kv' or 'q', got {bwd_payload!r}")
    kernels = kernels if kernels is not None else _default_kernels()
    offset = _offset(start_offset)
    if kernels.name == "cuda":
        check_qkv(q, k, v)
    if zigzag is None:
        zigzag = bool(causal) and world > 1
    N = q.shape[1]
    # zigzag hop classes start at chunk boundaries; the bf16 kernels need them 8-aligned
    unit = 2 * world * (8 if q.dtype == torch.bfloat16 else 1) if zigzag else world
    n_valid = None
    if N % unit:
        if not pad:
            raise ConfigError(f"gpus={world} does not divide seq={N}"
                              + (" into 2G chunks" if zigzag else "")
                              + "; enable pad to zero-fill the remainder")
        # RunConfig.pad / ring.partition(pad=True) (runner.py:96-98, ring.py:111-115)
        n_pad = -(-N // unit) * unit
        if zigzag and n_pad - N >= n_pad // unit:
            raise ConfigError(f"seq={N} too short to zero-pad into {unit} zigzag chunks")
        n_valid = N
        padz = lambda t: torch.cat([t, t.new_zeros(t.shape[0], n_pad - N, *t.shape[2:])], dim=1)
        q, k, v = padz(q), padz(k), padz(v)
        dout = padz(dout) if dout is not None else None
    scale = default_scale(q.shape[-1]) if softmax_scale is None else float(softmax_scale)
    # the reference applies the grid over the padded length n_total (ring.py:170, 233;
    # masking.py:48-63 cell bounds over `total`) and validates the real rows
    grid, causal = _bind_mask(mask, causal, q.shape[1], n_valid)
    shards = [[shard(t, r, world, zigzag) for r in range(world)] for t in (q, k, v)]
    do_sh = [shard(dout, r, world, zigzag) for r in range(world)] if dout is not None else None

    rec_f = [PassRecorder(r) for r in range(world)] if trace else [None] * world
    rec_b = [PassRecorder(r) for r in range(world)] if trace else [None] * world

    def one(rank, transport):
        qs, ks, vs = shards[0][rank], shards[1][rank], shards[2][rank]
        o, lse = ring_forward(qs, ks, vs, scale, causal, zigzag, transport, kernels, n_valid,
                              recorder=rec_f[rank], grid=grid, check=check, offset=offset)
        if do_sh is None:
            return o, lse, None
        bwd = ring_backward_qtravel if bwd_payload == "q" else ring_backward
        g = bwd(qs, ks, vs, o, lse, do_sh[rank], scale, causal, zigzag, transport, kernels,
                n_valid, recorder=rec_b[rank], grid=grid, check=check,
                deterministic=deterministic, offset=offset)
        return o, lse, g

    res = run_ranks(world, one, deadlock_timeout=deadlock_timeout)
    ptrace = None
    if trace:
        for rf, rb in zip(rec_f, rec_b):
            rf.ledger.elements_sent_backward = rb.ledger.elements_sent_backward
            rf.ledger.bytes_sent_backward = rb.ledger.bytes_sent_backward
            rf.ledger.ring_steps_backward = rb.ledger.ring_steps_backward
        ptrace = PassTrace(forward=merge(rec_f), backward=merge(rec_b) if do_sh else [],
                           ledgers=[rf.ledger for rf in rec_f])
    # _collect drops padded rows (sim.py:450-471)
    out = unshard([x[0] for x in res], zigzag, dim=1)[:, :N]
    lse = unshard([x[1] for x in res], zigzag, dim=2)[:, :, :N]
    if dout is None:
        return PassResult(out, lse, trace=ptrace)
    dq = unshard([x[2][0] for x in res], zigzag, dim=1)[:, :N]
    dk = unshard([x[2][1] for x in res], zigzag, dim=1)[:, :N]
    dv = unshard([x[2][2] for x in res], zigzag, dim=1)[:, :N]
    return PassResult(out, lse, dq, dk, dv, trace=ptrace)
