"""Ring hop schedule: sequence partition, global positions and hop classes.

Reference behaviour (pkg/src/burstsim):
  * device i holds contiguous row block i (ring.partition, ring.py:97-127);
  * at round r it holds the payload of origin (i - r) mod G (sim.py:565,
    ring.initial_forward_body ring.py:136-145);
  * causal = key position <= query position in GLOBAL coordinates
    (masking.py:116-117); a fully masked hop is skipped (ring.py:169-171).

B200 build (north star (4)): for causal runs the sequence is split into 2G
chunks of c = N/(2G) and rank i holds chunks i and 2G-1-i (zigzag), so every
rank does the same causal work.  With K/V from rank j at a hop:
  j == i : DIAG         causal inside both chunks (global positions)
  j <  i : K_EARLY_HALF all 2c queries x first key chunk (c keys), unmasked
  j >  i : Q_LATE_HALF  second query chunk (c rows) x all 2c keys, unmasked
Contiguous causal keeps the reference rule (FULL / DIAG / SKIP).
"""

from __future__ import annotations

from dataclasses import dataclass

FULL, DIAG, K_EARLY_HALF, Q_LATE_HALF, SKIP = "full", "diag", "k_early_half", "q_late_half", "skip"


@dataclass(frozen=True)
class PosMap:
    """Global position of local row i: i < seg_len ? pos0 + i : pos1 + (i - seg_len)."""
    pos0: int
    pos1: int
    seg_len: int

    def pos(self, i: int) -> int:
        return self.pos0 + i if i < self.seg_len else self.pos1 + (i - self.seg_len)

    def positions(self, n: int) -> list[int]:
        return [self.pos(i) for i in range(n)]


@dataclass(frozen=True)
class HopPlan:
    hop: int
    rank: int
    src: int            # origin rank of the visiting K/V block
    kind: str
    q_begin: int
    q_len: int
    k_begin: int
    k_len: int
    causal: bool        # element-level causal mask inside the rectangle
    q_map: PosMap
    k_map: PosMap
    grid: object = None  # masks.GridMask (bound) applied element-wise, or None
    key_order: object = None  # device int32 key-tile permutation (LAO forward), or None

    @property
    def skip(self) -> bool:
        return self.kind == SKIP

    def covers_all_queries(self, n_local: int) -> bool:
        return not self.skip and self.q_begin == 0 and self.q_len == n_local


def shard_map(rank: int, world: int, n_local: int, zigzag: bool) -> PosMap:
    """Global positions of the rows a rank holds."""
    if zigzag:
        if n_local % 2:
            raise ValueError("zigzag shards need an even local length")
        c = n_local // 2
        return PosMap(rank * c, (2 * world - 1 - rank) * c, c)
    return PosMap(rank * n_local, rank * n_local + n_local, n_local)


def source_rank(rank: int, world: int, hop: int, offset: int = 0) -> int:
    """Origin of the K/V block a rank holds at `hop` (sim.py:565, ring.py:143); a
    start offset rotates the initial assignment (initial_forward_body, ring.py:137-143:
    device i starts with block (i - offset) mod G)."""
    return (rank - offset - hop) % world


def valid_rows(rank: int, world: int, n_local: int, zigzag: bool, n_valid: int | None) -> int:
    """Rows of a (zero-padded) shard holding real positions < n_valid; always a
    prefix of the shard's local order (padding sits at the end of the sequence,
    ring.py:111-115 / _pad_rows 130-133)."""
    if n_valid is None:
        return n_local
    if not zigzag:
        return max(0, min(n_local, n_valid - rank * n_local))
    c = n_local // 2
    first = max(0, min(c, n_valid - rank * c))
    second = max(0, min(c, n_valid - (2 * world - 1 - rank) * c))
    return first + (second if first == c else 0)


def plan_hop(rank: int, world: int, hop: int, n_local: int, causal: bool,
             zigzag: bool, n_valid: int | None = None, grid=None, offset: int = 0) -> HopPlan:
    """Rectangle of one hop, with an optional block-sparse grid (masks.GridMask,
    bound to the global length): a rectangle whose every (query cell, key cell)
    pair is skipped becomes SKIP (BlockMask.decision, masking.py:79-106), any
    other keeps the grid for element-level masking in the kernels."""
    plan = _plan_hop(rank, world, hop, n_local, causal, zigzag, n_valid, offset)
    if grid is None or plan.skip:
        return plan
    qp = plan.q_map.positions(plan.q_begin + plan.q_len)[plan.q_begin:]
    kp = plan.k_map.positions(plan.k_begin + plan.k_len)[plan.k_begin:]
    if not qp or not kp:
        return plan
    qc = sorted({p // grid.qcell for p in qp})
    kc = sorted({p // grid.kcell for p in kp})
    if all((a, b) in grid.skip for a in qc for b in kc):
        return HopPlan(hop, rank, plan.src, SKIP, 0, 0, 0, 0, False, plan.q_map, plan.k_map)
    from dataclasses import replace
    return replace(plan, grid=grid)


def _plan_hop(rank: int, world: int, hop: int, n_local: int, causal: bool,
              zigzag: bool, n_valid: int | None = None, offset: int = 0) -> HopPlan:
    """Rectangle of one hop.  With padding (n_valid = real global length), padded
    keys are excluded by shortening the key range (BlockMask.with_padding,
    masking.py:74-75); under the causal rule they are invisible to every real
    query anyway, since they sit after all real positions."""
    src = source_rank(rank, world, hop, offset)
    qm = shard_map(rank, world, n_local, zigzag)
    km = shard_map(src, world, n_local, zigzag)
    n = n_local
    if not causal:
        kv = valid_rows(src, world, n_local, zigzag, n_valid)
        if kv == 0 and src != rank:
            return HopPlan(hop, rank, src, SKIP, 0, 0, 0, 0, False, qm, km)
        return HopPlan(hop, rank, src, FULL, 0, n, 0, kv, False, qm, km)
    if src == rank:
        return HopPlan(hop, rank, src, DIAG, 0, n, 0, n, True, qm, km)
    if zigzag:
        c = n // 2
        if src < rank:
            return HopPlan(hop, rank, src, K_EARLY_HALF, 0, n, 0, c, False, qm, km)
        return HopPlan(hop, rank, src, Q_LATE_HALF, c, c, 0, n, False, qm, km)
    if src < rank:
        return HopPlan(hop, rank, src, FULL, 0, n, 0, n, False, qm, km)
    return HopPlan(hop, rank, src, SKIP, 0, 0, 0, 0, False, qm, km)


def owner_of_contribution(rank: int, world: int, hop: int, offset: int = 0) -> int:
    """dK/dV computed at `hop` belong to the visiting block's home rank."""
    return source_rank(rank, world, hop, offset)


def contributor_to(rank: int, world: int, hop: int, offset: int = 0) -> int:
    """Rank that computed, at `hop`, a contribution for `rank`'s own block."""
    return (rank + offset + hop) % world


def hop_flops(plan: HopPlan, batch: int, heads: int, d: int) -> tuple[float, float]:
    """Algorithmic MMA FLOPs (fwd, bwd) of one hop (sim.py:80-87 model),
    counting only visible score entries for DIAG hops."""
    if plan.skip:
        return 0.0, 0.0
    if plan.grid is not None:
        area = _grid_area(plan)
    elif plan.causal:
        qp = plan.q_map.positions(plan.q_begin + plan.q_len)[plan.q_begin:]
        kp = plan.k_map.positions(plan.k_begin + plan.k_len)[plan.k_begin:]
        import bisect
        ks = sorted(kp)
        area = sum(bisect.bisect_right(ks, p) for p in qp)
    else:
        area = plan.q_len * plan.k_len
    f = 4.0 * batch * heads * area * d
    return f, 2.5 * f


def _grid_area(plan: HopPlan) -> int:
    """Visible (query, key) pairs of a hop under its grid mask (and causal rule),
    counted per grid cell (no N x N map)."""
    import numpy as np
    g = plan.grid
    qp = np.asarray(plan.q_map.positions(plan.q_begin + plan.q_len)[plan.q_begin:], dtype=np.int64)
    kp = np.asarray(plan.k_map.positions(plan.k_begin + plan.k_len)[plan.k_begin:], dtype=np.int64)
    qc = np.minimum(qp // g.qcell, g.n_query_blocks - 1)
    kc = np.minimum(kp // g.kcell, g.n_key_blocks - 1)
    open_ = (g.table() == 0).astype(np.int64)
    if not plan.causal:
        qn = np.bincount(qc, minlength=g.n_query_blocks)
        kn = np.bincount(kc, minlength=g.n_key_blocks)
        return int(qn @ open_ @ kn)
    area = 0
    for c in np.unique(kc):
        ks = np.sort(kp[kc == c])
        area += int((np.searchsorted(ks, qp, side="right") * open_[qc, c]).sum())
    return area


# ---------------------------------------------------------------------------
# shard helpers (torch tensors, sequence dim = 1 for [B, N, H, D])
# ---------------------------------------------------------------------------

def shard(x, rank: int, world: int, zigzag: bool, dim: int = 1):
    """Rows of the global tensor `x` that `rank` holds."""
    import torch
    n = x.shape[dim]
    if n % (2 * world if zigzag else world):
        raise ValueError(f"sequence length {n} not divisible for world={world} zigzag={zigzag}")
    if not zigzag:
        b = n // world
        return x.narrow(dim, rank * b, b).contiguous()
    c = n // (2 * world)
    return torch.cat([x.narrow(dim, rank * c, c), x.narrow(dim, (2 * world - 1 - rank) * c, c)],
                     dim=dim).contiguous()


def unshard(parts, zigzag: bool, dim: int = 1):
    """Inverse of `shard` given every rank's part in rank order."""
    import torch
    world = len(parts)
    if not zigzag:
        return torch.cat(list(parts), dim=dim)
    c = parts[0].shape[dim] // 2
    chunks = [None] * (2 * world)
    for r, p in enumerate(parts):
        chunks[r] = p.narrow(dim, 0, c)
        chunks[2 * world - 1 - r] = p.narrow(dim, c, c)
    return torch.cat(chunks, dim=dim)
