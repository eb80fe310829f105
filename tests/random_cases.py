"""Seeded random pass configurations (128) for the randomized parity sweep
(test_random_sweep.py): every option of run_ring_pass drawn together -- world size,
causal / zigzag, batch and heads, head dim and dtype, padding, a block-sparse grid,
backward payload, start offset, deterministic dQ -- so that combinations no
hand-written case names are covered too.  The checker is the dense fp64 oracle
(dense.py:63-118 restated in oracle/burst_oracle.py) over the global mask
(masking.py:79-130), so the sweep does not depend on the ring schedule it tests.
"""

from __future__ import annotations

import numpy as np


def _divisors(n, lo=1, hi=16):
    return [d for d in range(lo, hi + 1) if n % d == 0]


def draw_case(seed: int, large: bool = False) -> dict:
    r = np.random.default_rng(1000 + seed)
    f32 = r.random() < 0.25
    D = int(r.choice([16, 32, 64])) if f32 else int(r.choice([64, 128]))
    world = int(r.choice([1, 2, 3, 4, 5, 8]))
    causal = bool(r.random() < 0.5)
    zigzag = bool(causal and world > 1 and r.random() < 0.7)
    pad = bool(r.random() < 0.3)
    unit = 2 * world * (1 if f32 else 8) if zigzag else world
    lo, hi = (2048, 6144) if large else (96, 1200)
    n_total = unit * int(r.integers(max(1, lo // unit), max(2, hi // unit)))
    N = n_total
    if pad and unit > 1:
        # a length that is not a multiple of the unit; the pass zero-pads it to n_total,
        # the smallest multiple (api.run_ring_pass)
        # (zigzag: less than one chunk of padding, api.run_ring_pass's limit)
        gap = min(unit - 1, n_total // unit - 1) if zigzag else unit - 1
        N = n_total - int(r.integers(1, gap + 1)) if gap >= 1 else n_total
    pad = pad and N != n_total
    if not f32 and zigzag and (N // world // 2) % 8 and not pad:
        raise AssertionError("draw produced an unaligned zigzag chunk")
    mask = None
    if r.random() < 0.4:
        nqb = int(r.choice(_divisors(n_total, 2, 8) or [1]))
        nkb = int(r.choice(_divisors(n_total, 2, 8) or [1]))
        # never skip key column 0: position 0 is visible to every query (causal too),
        # so no row is left with nothing to attend to (MaskError)
        cells = [(a, b) for a in range(nqb) for b in range(1, nkb)]
        if cells:
            pick = r.choice(len(cells), size=int(r.integers(1, max(2, len(cells) // 2 + 1))),
                            replace=False)
            mask = {"n_query_blocks": nqb, "n_key_blocks": nkb,
                    "skip": [list(cells[i]) for i in sorted(pick)]}
    return {
        "seed": seed, "dtype": "f32" if f32 else "bf16", "D": D, "world": world,
        "causal": causal, "zigzag": zigzag, "pad": pad, "N": N, "n_total": n_total,
        "B": 1 if large else int(r.choice([1, 2])), "H": 1 if large else int(r.choice([1, 2, 3])),
        "payload": str(r.choice(["kv", "q"])),
        "offset": int(r.integers(0, world)) if world > 1 and r.random() < 0.4 else 0,
        "mask": mask,
        "deterministic": bool(not f32 and r.random() < 0.3),
    }


def dense_reference(q, k, v, do, case):
    """fp64 dense oracle per (batch, head) on the N valid rows: O, lse, dQ, dK, dV.
    The grid is bound to the padded length (ring.py:170, 233)."""
    from oracle import burst_oracle as orc
    B, N, H, D = q.shape
    grid = None
    if case["mask"] is not None:
        m = case["mask"]
        grid = orc.GridCells(m["n_query_blocks"], m["n_key_blocks"], m["skip"], case["n_total"])
    scale = D ** -0.5
    o, dq, dk, dv = (np.zeros((B, N, H, D)) for _ in range(4))
    lse = np.zeros((B, H, N))
    for b in range(B):
        for h in range(H):
            args = (q[b, :, h], k[b, :, h], v[b, :, h])
            o[b, :, h], lse[b, h] = orc.forward_dense(*args, scale, case["causal"], grid)
            dq[b, :, h], dk[b, :, h], dv[b, :, h] = orc.backward_dense(
                *args, do[b, :, h], scale, case["causal"], grid)
    return o, lse, dq, dk, dv


def pass_kwargs(case):
    return dict(causal=case["causal"], zigzag=case["zigzag"], pad=case["pad"],
                mask=case["mask"], bwd_payload=case["payload"], start_offset=case["offset"],
                deterministic=case["deterministic"])


CASES = [draw_case(s) for s in range(128)]   # the GPU sweep runs all
CPU_CASES = CASES[:32]                          # the host-logic sweep the first 32
# multi-tile lengths (2K-6K tokens, one head): long key-tile walks, odd tile counts per
# cluster pair, several query tiles per rank
LARGE_CASES = [draw_case(s, large=True) for s in range(500, 524)]
