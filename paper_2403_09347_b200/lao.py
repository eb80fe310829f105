"""LAO level: one attention rectangle on one device (no ring).

The reference's local-attention entry points (pkg/src/burstsim/local_attn.py) for a
query block against a key/value block, with global offsets for the causal rule:
  local_forward   = local_forward_tiled(...).finalize()   (local_attn.py:207-248, 127-135)
  local_backward  = local_backward(...)                   (local_attn.py:255-289)
over every (batch, head) slice of [batch, n, heads, head_dim] tensors, through the
same C ABI calls the ring uses (burst_lao_fwd / burst_lao_bwd).  The reference's
TileSpec is a CPU knob; the sm_100a kernels always use 128x128 tiles, so
`key_tile_order` permutes the hop's 128-key tiles.
"""

from __future__ import annotations

import torch

from .errors import ShapeError
from .kernels import CudaKernels, check_qkv, default_scale
from .schedule import DIAG, FULL, HopPlan, PosMap

KEY_TILE = 128

_kernels = None


def _kern() -> CudaKernels:
    global _kernels
    if _kernels is None:
        _kernels = CudaKernels()
    return _kernels


def _key_tile_order(order, n_k: int, device) -> torch.Tensor | None:
    """Device copy of a key-tile permutation, validated like local_attn.py:223-225."""
    if order is None:
        return None
    order = [int(i) for i in order]
    n_tiles = -(-n_k // KEY_TILE)
    if sorted(order) != list(range(n_tiles)):
        raise ShapeError(f"key_tile_order must permute range({n_tiles})")
    return torch.tensor(order, dtype=torch.int32, device=device)


def _plan(q, k, causal, row_offset, col_offset, mask, n_total, key_order=None) -> HopPlan:
    n_q, n_k = q.shape[1], k.shape[1]
    if row_offset < 0 or col_offset < 0:
        raise ShapeError("row_offset and col_offset must be non-negative")
    grid = None
    if mask is not None:
        from .api import _bind_mask
        total = n_total if n_total is not None else max(row_offset + n_q, col_offset + n_k)
        grid, causal = _bind_mask(mask, causal, total)
    return HopPlan(0, 0, 0, DIAG if causal else FULL, 0, n_q, 0, n_k, bool(causal),
                   PosMap(row_offset, row_offset + n_q, n_q),
                   PosMap(col_offset, col_offset + n_k, n_k), grid, key_order)


def local_forward(q, k, v, softmax_scale: float | None = None, causal: bool = False,
                  row_offset: int = 0, col_offset: int = 0, *, key_tile_order=None,
                  mask=None, n_total: int | None = None, check: str = "sync"):
    """Attention of a query block against one key/value block: (O, lse).

    q: [B, n_q, H, D], k/v: [B, n_k, H, D] (bf16 or f32, contiguous, on the GPU).
    `row_offset` / `col_offset`: global position of the first query / key row (the
    causal rule compares global positions, masking.py:116-117).  `key_tile_order`:
    visiting order of the 128-key tiles (a permutation of range(ceil(n_k / 128)));
    values agree with the default order to rounding.  `mask`: block-sparse grid
    (GridMask or spec) over a global span of `n_total` positions.
    Raises MaskError if a query row sees no key (PartialAttn.finalize)."""
    order = _key_tile_order(key_tile_order, k.shape[1], q.device)
    check_qkv(q, k, v)
    scale = default_scale(q.shape[-1]) if softmax_scale is None else float(softmax_scale)
    if not scale > 0:
        raise ShapeError(f"scale must be finite and positive, got {scale}")
    plan = _plan(q, k, causal, row_offset, col_offset, mask, n_total, order)
    kern = _kern()
    B, n, H, D = q.shape
    o = torch.empty_like(q)
    lse = torch.empty(B, H, n, dtype=torch.float32, device=q.device)
    state = kern.fwd_state(q, running=False)
    kern.fwd(plan, q, k, v, scale, state, o, lse, first=True, finalize=True)
    kern.finish(state, check, where="local_forward")
    return o, lse


def local_backward(q, k, v, dout, o, lse, softmax_scale: float | None = None,
                   causal: bool = False, row_offset: int = 0, col_offset: int = 0, *,
                   mask=None, n_total: int | None = None, deterministic: bool = False,
                   check: str = "sync"):
    """Gradient contributions (dQ, dK, dV) of one rectangle (local_attn.py:255-289).

    `o`, `lse`: this block's forward outputs (D = rowsum(dO * O) is formed on the
    device, ring.init_backward ring.py:195-218).  `deterministic`: dQ from the
    query-stationary kernel (one writer per row: bit-reproducible)."""
    check_qkv(q, k, v)
    if dout.shape != q.shape or o.shape != q.shape:
        raise ShapeError(f"dO and O must be {tuple(q.shape)}")
    if tuple(lse.shape) != (q.shape[0], q.shape[2], q.shape[1]):
        raise ShapeError("lse must be [batch, heads, n_q]")
    scale = default_scale(q.shape[-1]) if softmax_scale is None else float(softmax_scale)
    plan = _plan(q, k, causal, row_offset, col_offset, mask, n_total)
    kern = _kern()
    st = kern.bwd_prepare(o, dout.contiguous(), lse, deterministic=deterministic)
    dkp, dvp = kern.part(k), kern.part(v)
    kern.bwd(plan, q, k, v, dout.contiguous(), scale, st, dkp, dvp, accumulate=False)
    dq = torch.empty_like(q)
    dk, dv = torch.empty_like(k), torch.empty_like(v)
    # dq from the block's accumulator, dk/dv from the single contribution
    kern.tl_sum([st.dq_acc], dq, st.flags)
    kern.tl_sum([dkp], dk, st.flags)
    kern.tl_sum([dvp], dv, st.flags)
    kern.finish(st, check, where="local_backward")
    return dq, dk, dv

