"""CPU oracle for the BurstAttention hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference simulator's numerics
(`/root/reference/pkg/src/burstsim`, arXiv 2403.09347).  It exists so that the
GPU path can be checked against the reference's algorithm on the GPU box,
where `/root/reference` is absent.  Only `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s CPU-baseline leg may import it; the product package
`paper_2403_09347_b200` never does (and fails loudly without its CUDA library).

Parity of this restatement is PINNED against the reference itself: the golden
fixtures under `tests/golden/` were produced by importing the reference in
the dev container (`tests/golden/make_golden.py`), and
`tests/test_oracle_golden.py` checks every function here against them, plus
the reference's own known-answer tests (merge/finalize hand values).

Numerics contract, each function cites the line it
follows:
  * scores  S = (q * scale) @ k.T, queries scaled first  (local_attn.py:175)
  * masked scores are -inf before the row max           (local_attn.py:177-178)
  * m_eff = 0 for an all-masked row                       (local_attn.py:180)
  * merge uses exponent 0 where m == -inf                 (local_attn.py:113-116)
  * finalize: O = O_acc / l, lse = m + ln(l), MaskError if l == 0
                                                          (local_attn.py:127-135)
  * backward: P = exp(S - lse); dV += P^T dO; dP = dO V^T;
    dS = P * (dP - D); dQ += scale dS K; dK += scale dS^T Q
                                                          (local_attn.py:313-353)
  * D = rowsum(dO * O)                                    (ring.py:207)
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


# ---------------------------------------------------------------------------
# Error taxonomy (mirrors src/errors.py:4-33)
# ---------------------------------------------------------------------------

class OracleMaskError(ValueError):
    """A query row accumulated no unmasked key (local_attn.py:129-130)."""


class OracleNonFiniteError(FloatingPointError):
    """A result was NaN/Inf (local_attn.py:133-134)."""


# ---------------------------------------------------------------------------
# Masks: causal rule in GLOBAL positions (masking.py:110-130)
# ---------------------------------------------------------------------------

def causal_allowed(q_pos: np.ndarray, k_pos: np.ndarray) -> np.ndarray:
    """Element map, True where key position <= query position.

    Follows BlockMask.allowed (masking.py:116-117) but takes explicit global
    position vectors so that permuted (zigzag) shards can be checked.
    """
    return k_pos[None, :] <= q_pos[:, None]


class GridCells:
    """Coarse block grid over the global score matrix (BlockGrid, masking.py:33-63):
    n_query_blocks x n_key_blocks equal cells of a `total` x `total` matrix (validate
    requires divisibility, masking.py:135-139); `skip` = set of (qb, kb) cells whose
    scores are masked (allowed(), masking.py:120-128)."""

    def __init__(self, n_query_blocks, n_key_blocks, skip, total):
        self.nqb, self.nkb, self.total = int(n_query_blocks), int(n_key_blocks), int(total)
        self.skip = frozenset((int(a), int(b)) for a, b in skip)
        self.table = np.zeros((self.nqb, self.nkb), dtype=bool)
        for a, b in self.skip:
            self.table[a, b] = True

    def allowed(self, q_pos: np.ndarray, k_pos: np.ndarray) -> np.ndarray:
        qc = (np.asarray(q_pos) * self.nqb) // self.total
        kc = (np.asarray(k_pos) * self.nkb) // self.total
        return ~self.table[qc[:, None], kc[None, :]]


def mask_allowed(q_pos, k_pos, causal=False, grid=None):
    """Element map of the composed mask (BlockMask.allowed, masking.py:110-130) for
    explicit global positions, or None when nothing is masked."""
    out = None
    if causal:
        out = causal_allowed(np.asarray(q_pos), np.asarray(k_pos))
    if grid is not None:
        g = grid.allowed(q_pos, k_pos)
        out = g if out is None else (out & g)
    return out


# ---------------------------------------------------------------------------
# Partial (unnormalized) attention state -- PartialAttn (local_attn.py:66-135)
# ---------------------------------------------------------------------------

@dataclass
class Partial:
    o: np.ndarray   # rows x d, unnormalized output
    m: np.ndarray   # rows, running max (-inf until an unmasked entry is seen)
    l: np.ndarray   # rows, running exp-sum

    @classmethod
    def empty(cls, rows: int, d: int, dtype=np.float64) -> "Partial":
        # PartialAttn.empty, local_attn.py:82-91
        return cls(np.zeros((rows, d), dtype), np.full(rows, -np.inf, dtype),
                   np.zeros(rows, dtype))

    def merge(self, other: "Partial") -> "Partial":
        # PartialAttn.merge, local_attn.py:101-120
        dt = self.m.dtype
        m_new = np.maximum(self.m, other.m)
        with np.errstate(invalid="ignore"):
            fa = np.exp(np.where(np.isneginf(self.m), 0.0, self.m - m_new).astype(dt))
            fb = np.exp(np.where(np.isneginf(other.m), 0.0, other.m - m_new).astype(dt))
        self.l = fa * self.l + fb * other.l
        self.o = fa[:, None] * self.o + fb[:, None] * other.o
        self.m = m_new
        return self

    def finalize(self) -> tuple[np.ndarray, np.ndarray]:
        # PartialAttn.finalize, local_attn.py:127-135
        if np.any(self.l == 0):
            raise OracleMaskError("finalize: some query row accumulated no unmasked entries")
        o = self.o / self.l[:, None]
        lse = self.m + np.log(self.l)
        if not (np.isfinite(o).all() and np.isfinite(lse).all()):
            raise OracleNonFiniteError("finalize produced a non-finite value")
        return o, lse


def _block_partial(q, k, v, scale, allowed=None) -> Partial:
    # _block_partial, local_attn.py:171-190
    dt = q.dtype
    s = (q * dt.type(scale)) @ k.T
    if allowed is not None:
        s[~allowed] = -np.inf
    m = s.max(axis=1)
    m_eff = np.where(np.isneginf(m), 0.0, m).astype(dt)
    s = np.exp(s - m_eff[:, None])
    l = s.sum(axis=1)
    o = s @ v
    return Partial(o, m, l)


def local_forward_tiled(q, k, v, scale, tile_rows=128, tile_cols=128,
                        q_pos=None, k_pos=None, causal=False, grid=None,
                        key_tile_order=None) -> Partial:
    """LAO forward over one (query block x key block) rectangle.

    Restates local_forward_tiled (local_attn.py:207-248): query tiles x key
    tiles, each tile folded through the merge recurrence; a tile with no
    allowed entry is skipped (the SKIP decision, local_attn.py:151-155,
    masking.py:79-106).  ``q_pos``/``k_pos`` are global positions (the
    reference's row_offset/col_offset generalised to permuted shards).
    ``key_tile_order`` permutes the key-tile visits (local_attn.py:212-225).
    """
    dt = q.dtype
    rows, d = q.shape
    out = Partial.empty(rows, v.shape[1], dt)
    if causal or grid is not None:
        assert q_pos is not None and k_pos is not None
    k_edges = [(c0, min(c0 + tile_cols, k.shape[0])) for c0 in range(0, k.shape[0], tile_cols)]
    order = list(range(len(k_edges))) if key_tile_order is None else list(key_tile_order)
    if sorted(order) != list(range(len(k_edges))):
        raise ValueError(f"key_tile_order must permute range({len(k_edges)})")
    for r0 in range(0, rows, tile_rows):
        r1 = min(r0 + tile_rows, rows)
        acc = Partial.empty(r1 - r0, v.shape[1], dt)
        for idx in order:
            c0, c1 = k_edges[idx]
            allowed = None
            if causal or grid is not None:
                allowed = mask_allowed(q_pos[r0:r1], k_pos[c0:c1], causal, grid)
                if not allowed.any():
                    continue
                if allowed.all():
                    allowed = None
            acc.merge(_block_partial(q[r0:r1], k[c0:c1], v[c0:c1], scale, allowed))
        out.o[r0:r1], out.m[r0:r1], out.l[r0:r1] = acc.o, acc.m, acc.l
    return out


def local_backward(q, k, v, do, lse, d_stat, scale, tile_rows=128, tile_cols=128,
                   q_pos=None, k_pos=None, causal=False, grid=None):
    """Gradient contributions of one rectangle (local_attn.py:255-289, tiled
    form _backward_tiled 313-353).  Returns (dQ, dK, dV) contributions."""
    dt = q.dtype
    sc = dt.type(scale)
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    for r0 in range(0, q.shape[0], tile_rows):
        r1 = min(r0 + tile_rows, q.shape[0])
        for c0 in range(0, k.shape[0], tile_cols):
            c1 = min(c0 + tile_cols, k.shape[0])
            allowed = None
            if causal or grid is not None:
                allowed = mask_allowed(q_pos[r0:r1], k_pos[c0:c1], causal, grid)
                if not allowed.any():
                    continue
            s = (q[r0:r1] * sc) @ k[c0:c1].T
            if allowed is not None:
                s[~allowed] = -np.inf
            p = np.exp(s - lse[r0:r1, None])
            dv[c0:c1] += p.T @ do[r0:r1]
            dp = do[r0:r1] @ v[c0:c1].T
            ds = p * (dp - d_stat[r0:r1, None])
            dq[r0:r1] += (ds @ k[c0:c1]) * sc
            dk[c0:c1] += (ds.T @ q[r0:r1]) * sc
    for name, g in (("dQ", dq), ("dK", dk), ("dV", dv)):
        if not np.isfinite(g).all():
            raise OracleNonFiniteError(f"local backward produced non-finite {name}")
    return dq, dk, dv


# ---------------------------------------------------------------------------
# Dense oracle (dense.py:63-118)
# ---------------------------------------------------------------------------

def forward_dense(q, k, v, scale, causal=False, grid=None):
    # _forward_arrays, dense.py:70-87
    s = (q * q.dtype.type(scale)) @ k.T
    allowed = mask_allowed(np.arange(q.shape[0]), np.arange(k.shape[0]), causal, grid)
    if allowed is not None:
        s[~allowed] = -np.inf
    m = s.max(axis=1)
    m_eff = np.where(np.isneginf(m), 0.0, m).astype(s.dtype)
    p = np.exp(s - m_eff[:, None])
    l = p.sum(axis=1)
    if np.any(l == 0):
        raise OracleMaskError("softmax row with no unmasked entries")
    o = (p @ v) / l[:, None]
    lse = m + np.log(l)
    return o, lse


def backward_dense(q, k, v, do, scale, causal=False, grid=None):
    # backward_dense, dense.py:99-118
    o, lse = forward_dense(q, k, v, scale, causal, grid)
    s = (q * q.dtype.type(scale)) @ k.T
    allowed = mask_allowed(np.arange(q.shape[0]), np.arange(k.shape[0]), causal, grid)
    if allowed is not None:
        s[~allowed] = -np.inf
    prob = np.exp(s - lse[:, None])
    d_stat = (do * o).sum(axis=1)
    dv = prob.T @ do
    dp = do @ v.T
    ds = prob * (dp - d_stat[:, None])
    sc = q.dtype.type(scale)
    return (ds @ k) * sc, (ds.T @ q) * sc, dv


# ---------------------------------------------------------------------------
# Ring pass (ring.py:97-242, sim.py:501-657 lockstep executor)
# ---------------------------------------------------------------------------

def contiguous_positions(n: int, G: int) -> list[np.ndarray]:
    """partition (ring.py:97-127): device i holds rows [i*n/G, (i+1)*n/G)."""
    b = n // G
    return [np.arange(i * b, (i + 1) * b) for i in range(G)]


def zigzag_positions(n: int, G: int) -> list[np.ndarray]:
    """Load-balanced causal partition (north star (4); not in the reference).

    Split N into 2G chunks of c = N/(2G); rank i holds chunks i and 2G-1-i.
    The causal rule stays the reference's global-position rule
    (masking.py:116-117), so parity is checked after un-permuting.
    """
    c = n // (2 * G)
    return [np.concatenate([np.arange(i * c, (i + 1) * c),
                            np.arange((2 * G - 1 - i) * c, (2 * G - i) * c)])
            for i in range(G)]


def ring_forward(q, k, v, scale, G, causal=False, zigzag=False, tile=128, grid=None):
    """Lockstep ring forward (sim.py:551-574 + ring.forward_step 158-181).

    Device i holds payload from origin (i - r) mod G at round r (sim.py:565,
    ring.py:143).  Returns per-device (positions, O, lse).
    """
    n = q.shape[0]
    pos = zigzag_positions(n, G) if zigzag else contiguous_positions(n, G)
    states = [Partial.empty(len(p), v.shape[1], q.dtype) for p in pos]
    for r in range(G):
        for i in range(G):
            j = (i - r) % G
            qp, kp = pos[i], pos[j]
            allowed = mask_allowed(qp, kp, causal, grid)
            if allowed is not None and not allowed.any():
                continue  # whole-hop SKIP (ring.py:169-171)
            part = local_forward_tiled(q[qp], k[kp], v[kp], scale, tile, tile,
                                       qp, kp, causal, grid)
            states[i].merge(part)   # hop merge (ring.py:180)
    outs = []
    for i in range(G):
        o, lse = states[i].finalize()   # finalize_forward (ring.py:184-188)
        outs.append((pos[i], o, lse))
    return outs


def ring_backward(q, k, v, do, scale, G, causal=False, zigzag=False, tile=128, grid=None):
    """Lockstep ring backward (ring.init_backward 195-218, backward_step 221-242).

    Returns global (dQ, dK, dV, O, lse) assembled from all devices.
    """
    n = q.shape[0]
    pos = zigzag_positions(n, G) if zigzag else contiguous_positions(n, G)
    fwd = ring_forward(q, k, v, scale, G, causal, zigzag, tile, grid)
    o = np.zeros_like(q)
    lse = np.zeros(n, q.dtype)
    for p, oi, li in fwd:
        o[p], lse[p] = oi, li
    d_stat = (do * o).sum(axis=1)          # ring.py:207
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    for r in range(G):
        for i in range(G):
            j = (i - r) % G
            qp, kp = pos[i], pos[j]
            allowed = mask_allowed(qp, kp, causal, grid)
            if allowed is not None and not allowed.any():
                continue
            a, b, c = local_backward(q[qp], k[kp], v[kp], do[qp], lse[qp], d_stat[qp],
                                     scale, tile, tile, qp, kp, causal, grid)
            dq[qp] += a
            dk[kp] += b
            dv[kp] += c
    return dq, dk, dv, o, lse


# ---------------------------------------------------------------------------
# Inputs (runner.generate_inputs, runner.py:144-162)
# ---------------------------------------------------------------------------

def generate_inputs(seq: int, dim: int, heads: int, batch: int = 1, seed: int = 0,
                    dtype=np.float32):
    """Q, K, V, dO of shape (batch*heads, seq, dim): four independent Philox
    streams spawned from SeedSequence(seed), N(0,1) draws, scale d^-0.5."""
    children = np.random.SeedSequence(seed).spawn(4)
    streams = [np.random.Generator(np.random.Philox(c)) for c in children]
    raw = [g.standard_normal((batch * heads, seq, dim)).astype(dtype) for g in streams]
    return raw[0], raw[1], raw[2], raw[3], float(dim) ** -0.5


# ---------------------------------------------------------------------------
# FLOP model (sim.py:80-87)
# ---------------------------------------------------------------------------

def attn_flops(batch: int, heads: int, n_q: int, n_k: int, d: int,
               causal: bool = False) -> tuple[float, float]:
    """Algorithmic (MMA) FLOPs: fwd 4*r*c*d, bwd 10*r*c*d (sim.py:80-87),
    halved for causal.  Returns (forward, backward)."""
    f = 4.0 * batch * heads * n_q * n_k * d
    b = 10.0 * batch * heads * n_q * n_k * d
    if causal:
        f, b = f / 2, b / 2
    return f, b


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float32 (identical
    bf16-rounded inputs for both sides of a parity check)."""
    a = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((a >> 16) & 1) + 0x7FFF
    return ((a + r) & 0xFFFF0000).view(np.float32)


LN2 = math.log(2.0)
