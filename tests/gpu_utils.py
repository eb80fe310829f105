"""Helpers shared by the GPU parity tests (the oracle is the checker)."""

from __future__ import annotations

import numpy as np
import torch

from oracle import burst_oracle as orc


def make_inputs(B, N, H, D, seed=0, dtype=torch.bfloat16, device="cuda"):
    """Seeded N(0,1) q, k, v, dO [B, N, H, D] (runner.generate_inputs distribution)."""
    g = torch.Generator().manual_seed(seed)
    ts = [torch.randn(B, N, H, D, generator=g) for _ in range(4)]
    return [t.to(dtype).to(device) for t in ts]


def oracle_ring(q, k, v, do, world, causal, zigzag, scale=None, tile=128, with_grad=True):
    """Run the numpy oracle per (b, h) slice on the SAME (rounded) inputs.

    Returns numpy arrays o [B,N,H,D], lse [B,H,N], dq, dk, dv.
    """
    B, N, H, D = q.shape
    scale = D ** -0.5 if scale is None else scale
    f = lambda t: t.float().cpu().numpy().astype(np.float64)
    qn, kn, vn, dn = f(q), f(k), f(v), f(do) if do is not None else None
    o = np.zeros((B, N, H, D))
    lse = np.zeros((B, H, N))
    dq, dk, dv = np.zeros_like(o), np.zeros_like(o), np.zeros_like(o)
    for b in range(B):
        for h in range(H):
            if with_grad:
                a, bb, c, oo, ll = orc.ring_backward(qn[b, :, h], kn[b, :, h], vn[b, :, h],
                                                     dn[b, :, h], scale, world, causal, zigzag,
                                                     tile)
                dq[b, :, h], dk[b, :, h], dv[b, :, h] = a, bb, c
            else:
                outs = orc.ring_forward(qn[b, :, h], kn[b, :, h], vn[b, :, h], scale, world,
                                        causal, zigzag, tile)
                oo = np.zeros((N, D))
                ll = np.zeros(N)
                for p, oi, li in outs:
                    oo[p], ll[p] = oi, li
            o[b, :, h], lse[b, h] = oo, ll
    return o, lse, dq, dk, dv


def max_abs(a, b):
    a = a.detach().float().cpu().numpy() if isinstance(a, torch.Tensor) else a
    return float(np.max(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64))))


def rel_err(a, b):
    """Per-tensor max|x - ref| / max|ref| (SURVEY.md 8(c) definition)."""
    b = np.asarray(b, np.float64)
    return max_abs(a, b) / max(float(np.max(np.abs(b))), 1e-30)


def poison_allocator(nbytes=256 << 20):
    """Fill, then free, a large block so the caching allocator hands out NaN-filled
    memory to the next torch.empty calls: any buffer a kernel forgets to define
    then shows up as NaN in the results instead of passing by luck."""
    x = torch.full((nbytes // 4,), float("nan"), dtype=torch.float32, device="cuda")
    del x
