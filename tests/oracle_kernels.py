"""Oracle-backed kernel provider for HOST-LOGIC tests only (CPU tensors).

Implements the same interface as paper_2403_09347_b200.kernels.CudaKernels
with the numpy oracle, so the ring engine (schedule, transports, K/V rotation,
dK/dV routing, finalisation) can be exercised on CPU with gloo.  It is
injected explicitly by tests; the product never imports it.
"""

from __future__ import annotations

import numpy as np
import torch

from oracle import burst_oracle as orc


def _np(t):
    return t.detach().double().cpu().numpy()


def _grid(plan):
    """The product's GridMask as the oracle's GridCells (same BlockGrid semantics)."""
    g = plan.grid
    if g is None:
        return None
    return orc.GridCells(g.n_query_blocks, g.n_key_blocks, g.skip, g.total)


class OracleKernels:
    name = "oracle"

    def __init__(self):
        self.launches = 0

    def fwd_state(self, q, running=True):
        # undefined until a first hop writes it, like the CUDA state (torch.empty)
        B, n, H, D = q.shape
        return {"o": np.full((B, H, n, D), np.nan), "m": np.full((B, H, n), np.nan),
                "l": np.full((B, H, n), np.nan)}

    def fwd_init(self, state, stream=None):
        state["o"][:] = 0.0
        state["m"][:] = -np.inf
        state["l"][:] = 0.0

    def finish(self, state, check, stream=None, where="BurstAttention"):
        """The oracle raises its errors synchronously (MaskError / NonFiniteError)."""

    def accumulate(self, acc_pair, part_pair, like, stream=None):
        for a, p in zip(acc_pair, part_pair):
            a += p

    def part(self, k):
        return torch.zeros(k.shape, dtype=torch.float64)

    def fwd(self, plan, q, k, v, scale, state, o, lse, first, finalize, stream=None):
        self.launches += 1
        B, n, H, D = q.shape
        qn, kn, vn = _np(q), _np(k), _np(v)
        qp = np.array(plan.q_map.positions(n))
        kp = np.array(plan.k_map.positions(k.shape[1]))
        qs = slice(plan.q_begin, plan.q_begin + plan.q_len)
        ks = slice(plan.k_begin, plan.k_begin + plan.k_len)
        for b in range(B):
            for h in range(H):
                part = orc.local_forward_tiled(qn[b, qs, h], kn[b, ks, h], vn[b, ks, h], scale,
                                               128, 128, qp[qs], kp[ks], plan.causal,
                                               _grid(plan))
                if first:
                    acc = part
                else:
                    acc = orc.Partial(state["o"][b, h, qs].copy(), state["m"][b, h, qs].copy(),
                                      state["l"][b, h, qs].copy())
                    acc.merge(part)
                if finalize:
                    oo, ll = acc.finalize()
                    o[b, qs, h] = torch.from_numpy(oo).to(o.dtype)
                    lse[b, h, qs] = torch.from_numpy(ll).to(lse.dtype)
                else:
                    state["o"][b, h, qs], state["m"][b, h, qs], state["l"][b, h, qs] = \
                        acc.o, acc.m, acc.l

    def fwd_finalize(self, state, o, lse, stream=None):
        self.launches += 1
        B, n, H, D = o.shape
        for b in range(B):
            for h in range(H):
                oo, ll = orc.Partial(state["o"][b, h], state["m"][b, h], state["l"][b, h]).finalize()
                o[b, :, h] = torch.from_numpy(oo).to(o.dtype)
                lse[b, h] = torch.from_numpy(ll).to(lse.dtype)

    def bwd_prepare(self, o, dout, lse, stream=None, deterministic=False):
        self.launches += 1
        d_stat = (_np(o) * _np(dout)).sum(-1).transpose(0, 2, 1)   # [B, H, n]
        return {"lse": _np(lse), "D": d_stat, "dq": np.zeros(tuple(o.shape))}

    def bwd(self, plan, q, k, v, dout, scale, st, dk_part, dv_part, accumulate, stream=None):
        self.launches += 1
        B, n, H, D = q.shape
        qn, kn, vn, dn = _np(q), _np(k), _np(v), _np(dout)
        qp = np.array(plan.q_map.positions(n))
        kp = np.array(plan.k_map.positions(k.shape[1]))
        qs = slice(plan.q_begin, plan.q_begin + plan.q_len)
        ks = slice(plan.k_begin, plan.k_begin + plan.k_len)
        if not accumulate:
            dk_part.zero_()
            dv_part.zero_()
        for b in range(B):
            for h in range(H):
                dq, dk, dv = orc.local_backward(qn[b, qs, h], kn[b, ks, h], vn[b, ks, h],
                                                dn[b, qs, h], st["lse"][b, h, qs],
                                                st["D"][b, h, qs], scale, 128, 128, qp[qs],
                                                kp[ks], plan.causal, _grid(plan))
                st["dq"][b, qs, h] += dq
                dk_part[b, ks, h] += torch.from_numpy(dk)
                dv_part[b, ks, h] += torch.from_numpy(dv)

    def bwd_finalize(self, st, dk_parts, dv_parts, dq, dk, dv, stream=None):
        self.launches += 1
        dq.copy_(torch.from_numpy(st["dq"]).to(dq.dtype))
        dk.copy_(sum(p for p in dk_parts).to(dk.dtype))
        dv.copy_(sum(p for p in dv_parts).to(dv.dtype))

    # travelling-query backward (f2)
    def stats_tensors(self, st):
        return [torch.from_numpy(st["lse"].copy()), torch.from_numpy(st["D"].copy())]

    def visiting_state(self, st, stats, dq_part):
        return {"lse": stats[0].numpy(), "D": stats[1].numpy(), "dq": dq_part.numpy()}

    def dq_part(self, q, stream=None, reuse=None):
        if reuse is not None:
            reuse.zero_()
            return reuse
        return torch.zeros(tuple(q.shape), dtype=torch.float64)

    def dq_like(self, q):
        return torch.empty(tuple(q.shape), dtype=torch.float64, device="meta")

    def accumulate_dq(self, st, part, like, stream=None):
        st["dq"] += part.numpy()

    def bwd_finalize_qtravel(self, st, dq_parts, dk_acc, dv_acc, dq, dk, dv, stream=None):
        self.launches += 1
        tot = torch.from_numpy(st["dq"]) + sum((p for p in dq_parts), torch.zeros(tuple(dq.shape),
                                                                                  dtype=torch.float64))
        dq.copy_(tot.to(dq.dtype))
        dk.copy_(dk_acc.to(dk.dtype))
        dv.copy_(dv_acc.to(dv.dtype))

    def zero_(self, bufs, stream=None):
        for b in bufs:
            b.zero_()
