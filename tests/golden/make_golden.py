"""Generate golden vectors by running the REFERENCE itself (dev container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the unmodified reference simulator (`burstsim`, /root/reference/pkg/src)
and records its outputs for a set of small cases plus the BASELINE C1 config.
The GPU box has no /root/reference, so the fixtures are committed; the oracle
(`oracle/burst_oracle.py`) is pinned against them by tests/test_oracle_golden.py.
Inputs are NOT stored: they are regenerated from the seed with the reference's
generator (runner.generate_inputs, runner.py:144-162), and a checksum of the
reference's inputs is stored to prove the regeneration matches.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from burstsim import ring  # noqa: E402
from burstsim.dense import AttnProblem, backward_dense, forward_dense  # noqa: E402
from burstsim.linalg import Matrix, Vector  # noqa: E402
from burstsim.local_attn import TileSpec, local_backward, local_forward_tiled  # noqa: E402
from burstsim.masking import BlockMask  # noqa: E402
from burstsim.runner import RunConfig, generate_inputs  # noqa: E402
from burstsim.sim import build_cluster, run_ring_pass  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def _checksum(arrs):
    return np.array([float(np.sum(a.astype(np.float64))) for a in arrs] +
                    [float(a.reshape(-1)[7]) for a in arrs])


def ring_case(name, seq, dim, heads, gpus, precision, mask=None, tile=None, seed=0, pad=False):
    cfg = RunConfig(seq=seq, dim=dim, heads=heads, gpus=gpus, precision=precision,
                    mask=mask, tile_rows=tile, seed=seed, pad=pad)
    cfg.validate()
    problems, do = generate_inputs(cfg)
    tiles = TileSpec(tile, tile) if tile else None
    cluster = build_cluster(problems, gpus, tiles, pad=pad)
    fwd = run_ring_pass(cluster, "forward")
    bwd = run_ring_pass(cluster, "backward", do_slices=do)
    out = {}
    out["o"] = np.stack([o.array for o, _ in fwd.outputs])
    out["lse"] = np.stack([l.array for _, l in fwd.outputs])
    out["dq"] = np.stack([g[0].array for g in bwd.grads])
    out["dk"] = np.stack([g[1].array for g in bwd.grads])
    out["dv"] = np.stack([g[2].array for g in bwd.grads])
    q = np.stack([p.Q.array for p in problems])
    k = np.stack([p.K.array for p in problems])
    v = np.stack([p.V.array for p in problems])
    g = np.stack([m.array for m in do])
    out["input_checksum"] = _checksum([q, k, v, g])
    is_causal = mask == "causal" or (isinstance(mask, dict) and bool(mask.get("causal")))
    out["meta"] = np.array([seq, dim, heads, gpus, seed, 1 if is_causal else 0,
                            tile or 0, 1 if precision == "single" else 2])
    if isinstance(mask, dict):     # block-sparse grid (BlockGrid, masking.py:33-63)
        out["grid"] = np.array([mask["n_query_blocks"], mask["n_key_blocks"]])
        out["grid_skip"] = np.array(mask["skip"], dtype=np.int64).reshape(-1, 2)
    # dense oracle on the same inputs, for the tolerance the reference accepts
    if seq <= 256:
        dq = [backward_dense(p, m) for p, m in zip(problems, do)]
        out["dense_o"] = np.stack([forward_dense(p).O.array for p in problems])
        out["dense_dq"] = np.stack([x[0].array for x in dq])
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print("wrote", name, {k: v.shape for k, v in out.items()})


def lao_case(name, rows, cols, dim, row_offset, col_offset, n_total, causal, seed):
    """local_forward_tiled / local_backward on one rectangle in global coords."""
    rng = np.random.Generator(np.random.Philox(seed))
    q, k, v, do = (rng.standard_normal((r, dim)) for r in (rows, cols, cols, rows))
    mask = BlockMask(causal=True) if causal else None
    part = local_forward_tiled(Matrix.from_array(q), Matrix.from_array(k),
                               Matrix.from_array(v), dim ** -0.5, TileSpec(4, 4), mask,
                               row_offset=row_offset, col_offset=col_offset,
                               n_total=n_total)
    lse = rng.standard_normal(rows) + 3.0
    dst = rng.standard_normal(rows)
    dq, dk, dv = local_backward(Matrix.from_array(q), Matrix.from_array(k),
                                Matrix.from_array(v), Matrix.from_array(do),
                                Vector(lse), Vector(dst), dim ** -0.5, TileSpec(4, 4),
                                mask, row_offset=row_offset, col_offset=col_offset,
                                n_total=n_total)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"),
                        q=q, k=k, v=v, do=do, lse_in=lse, d_in=dst,
                        o=part.o, m=part.m, l=part.l,
                        dq=dq.array, dk=dk.array, dv=dv.array,
                        meta=np.array([rows, cols, dim, row_offset, col_offset,
                                       n_total, int(causal), seed]))
    print("wrote", name)


def order_case(name, rows, cols, dim, row_offset, col_offset, n_total, causal, seed, order):
    """local_forward_tiled with a permuted key-tile order (key_tile_order,
    local_attn.py:212-225), 128x128 tiles (the GPU kernels' tile)."""
    rng = np.random.Generator(np.random.Philox(seed))
    q, k, v = (rng.standard_normal((r, dim)) for r in (rows, cols, cols))
    mask = BlockMask(causal=True) if causal else None
    part = local_forward_tiled(Matrix.from_array(q), Matrix.from_array(k),
                               Matrix.from_array(v), dim ** -0.5, TileSpec(128, 128), mask,
                               row_offset=row_offset, col_offset=col_offset,
                               n_total=n_total, key_tile_order=list(order))
    o, lse = part.finalize()
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), q=q, k=k, v=v,
                        o=o.array, lse=lse.array, order=np.array(order),
                        meta=np.array([rows, cols, dim, row_offset, col_offset, n_total,
                                       int(causal), seed]))
    print("wrote", name)


def grid_cases():
    """Block-sparse grid masks through the whole ring (mask_from_spec dict form,
    masking.py:150-180), with and without the causal constraint."""
    ring_case("ring_n64_d16_h2_g4_grid_f64", 64, 16, 2, 4, "double",
              mask={"n_query_blocks": 4, "n_key_blocks": 4,
                    "skip": [[0, 3], [2, 1], [1, 1], [3, 0]]}, tile=8, seed=11)
    ring_case("ring_n128_d16_h1_g4_grid_causal_f64", 128, 16, 1, 4, "double",
              mask={"n_query_blocks": 8, "n_key_blocks": 8, "causal": True,
                    "skip": [[3, 1], [5, 2], [7, 0], [6, 6], [2, 0]]}, tile=16, seed=12)
    ring_case("ring_n256_d32_h1_g2_grid_causal_f32", 256, 32, 1, 2, "single",
              mask={"n_query_blocks": 4, "n_key_blocks": 4, "causal": True,
                    "skip": [[1, 0], [3, 2]]}, tile=64, seed=13)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "grid":
        grid_cases()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "order":
        order_case("lao_order_r256_c640_d64_causal", 256, 640, 64, 512, 0, 768, True, 21,
                   [3, 0, 4, 2, 1])
        sys.exit(0)
    # BASELINE.json configs[0]: seq 1024, d 64, 2 heads, G 2, fp32, non-causal.
    # 128x128 tiles (the default SRAM tile gives identical math, 100x slower).
    ring_case("c1_seq1024_d64_h2_g2_f32", 1024, 64, 2, 2, "single", tile=128)
    # small fp64 rings: non-causal and causal (contiguous partition, whole-hop skip)
    ring_case("ring_n64_d16_h2_g4_f64", 64, 16, 2, 4, "double", tile=8, seed=1)
    ring_case("ring_n64_d16_h1_g4_causal_f64", 64, 16, 1, 4, "double", mask="causal",
              tile=8, seed=2)
    ring_case("ring_n256_d64_h1_g2_causal_f32", 256, 64, 1, 2, "single", mask="causal",
              tile=64, seed=3)
    # padding: seq not divisible by G (RunConfig.pad, ring.partition pad=True)
    ring_case("ring_n100_d16_h2_g3_pad_f32", 100, 16, 2, 3, "single", tile=16, seed=4, pad=True)
    ring_case("ring_n98_d16_h1_g4_causal_pad_f32", 98, 16, 1, 4, "single", mask="causal",
              tile=16, seed=5, pad=True)
    # LAO rectangles in global coordinates (row/col offsets), causal partial tiles
    lao_case("lao_r12_c20_d8_causal", 12, 20, 8, 16, 4, 40, True, 7)
    lao_case("lao_r16_c16_d8_full", 16, 16, 8, 0, 16, 32, False, 8)
    grid_cases()
    order_case("lao_order_r256_c640_d64_causal", 256, 640, 64, 512, 0, 768, True, 21,
               [3, 0, 4, 2, 1])
