"""Pin the CPU oracle against the reference's own outputs and known answers.

The fixtures were produced by running the unmodified reference simulator
(tests/golden/make_golden.py); here the restatement in oracle/ must reproduce
them.  Known-answer tests mirror pkg/tests/test_local_attn.py:18-83.
"""

import math

import numpy as np
import pytest

from oracle import burst_oracle as orc


def test_merge_hand_value():
    # pkg/tests/test_local_attn.py:18-29
    a = orc.Partial(o=np.array([[2.0]]), m=np.array([1.0]), l=np.array([2.0]))
    b = orc.Partial(o=np.array([[8.0]]), m=np.array([3.0]), l=np.array([4.0]))
    a.merge(b)
    assert a.m[0] == 3.0
    assert a.l[0] == pytest.approx(4.270670566473225, abs=1e-15)
    assert a.o[0, 0] == pytest.approx(2.0 * math.exp(-2.0) + 8.0, abs=1e-14)


def test_merge_with_empty_is_passthrough():
    # pkg/tests/test_local_attn.py:31-41
    rng = np.random.default_rng(0)
    o, m, l = rng.standard_normal((3, 2)), rng.standard_normal(3), np.abs(rng.standard_normal(3)) + .5
    s = orc.Partial.empty(3, 2)
    s.merge(orc.Partial(o.copy(), m.copy(), l.copy()))
    assert np.array_equal(s.o, o) and np.array_equal(s.m, m) and np.array_equal(s.l, l)


def test_finalize_hand_value_and_unvisited_rows():
    # pkg/tests/test_local_attn.py:74-83
    o, lse = orc.Partial(np.array([[6.0, 9.0]]), np.array([0.0]), np.array([3.0])).finalize()
    assert np.allclose(o, [[2.0, 3.0]]) and lse[0] == pytest.approx(math.log(3.0))
    with pytest.raises(orc.OracleMaskError):
        orc.Partial.empty(2, 2).finalize()


@pytest.mark.parametrize("name,tol", [
    ("c1_seq1024_d64_h2_g2_f32", 2e-6),
    ("ring_n64_d16_h2_g4_f64", 1e-12),
    ("ring_n64_d16_h1_g4_causal_f64", 1e-12),
    ("ring_n256_d64_h1_g2_causal_f32", 2e-6),
    ("ring_n64_d16_h2_g4_grid_f64", 1e-12),
    ("ring_n128_d16_h1_g4_grid_causal_f64", 1e-12),
    ("ring_n256_d32_h1_g2_grid_causal_f32", 2e-6),
])
def test_oracle_ring_matches_reference(golden, name, tol):
    g = golden(name)
    seq, dim, heads, gpus, seed, causal, tile, prec = (int(x) for x in g["meta"])
    dt = np.float32 if prec == 1 else np.float64
    q, k, v, do, scale = orc.generate_inputs(seq, dim, heads, 1, seed, dt)
    # the regenerated inputs are the reference's inputs
    cs = np.array([float(np.sum(a.astype(np.float64))) for a in (q, k, v, do)] +
                  [float(a.reshape(-1)[7]) for a in (q, k, v, do)])
    assert np.array_equal(cs, g["input_checksum"])
    grid = None
    if "grid" in g:   # block-sparse grid mask (BlockGrid, masking.py:33-63)
        grid = orc.GridCells(g["grid"][0], g["grid"][1], g["grid_skip"].tolist(), seq)
    for s in range(heads):
        dq, dk, dv, o, lse = orc.ring_backward(q[s], k[s], v[s], do[s], scale, gpus,
                                               causal=bool(causal), tile=tile, grid=grid)
        for key, got in (("o", o), ("lse", lse), ("dq", dq), ("dk", dk), ("dv", dv)):
            ref = g[key][s]
            err = np.max(np.abs(got.astype(np.float64) - ref)) / max(np.max(np.abs(ref)), 1e-30)
            assert err < tol, (name, key, err)


def test_oracle_zigzag_matches_reference_dense(golden):
    # Zigzag is not in the reference; its causal answer must equal the
    # reference's dense causal oracle on the same inputs.
    g = golden("ring_n64_d16_h1_g4_causal_f64")
    q, k, v, do, scale = orc.generate_inputs(64, 16, 1, 1, 2, np.float64)
    dq, dk, dv, o, lse = orc.ring_backward(q[0], k[0], v[0], do[0], scale, 4,
                                           causal=True, zigzag=True, tile=8)
    assert np.max(np.abs(o - g["dense_o"][0])) < 1e-12
    assert np.max(np.abs(dq - g["dense_dq"][0])) < 1e-11
    assert np.max(np.abs(dk - g["dk"][0])) < 1e-11
    assert np.max(np.abs(dv - g["dv"][0])) < 1e-11


@pytest.mark.parametrize("name", ["lao_r12_c20_d8_causal", "lao_r16_c16_d8_full"])
def test_oracle_lao_matches_reference(golden, name):
    g = golden(name)
    rows, cols, dim, r0, c0, n_total, causal, seed = (int(x) for x in g["meta"])
    qp, kp = np.arange(r0, r0 + rows), np.arange(c0, c0 + cols)
    part = orc.local_forward_tiled(g["q"], g["k"], g["v"], dim ** -0.5, 4, 4, qp, kp,
                                   bool(causal))
    assert np.allclose(part.o, g["o"], atol=1e-12, rtol=0)
    assert np.array_equal(np.isneginf(part.m), np.isneginf(g["m"]))
    fin = ~np.isneginf(g["m"])
    assert np.allclose(part.m[fin], g["m"][fin], atol=1e-13)
    assert np.allclose(part.l, g["l"], atol=1e-12)
    dq, dk, dv = orc.local_backward(g["q"], g["k"], g["v"], g["do"], g["lse_in"],
                                    g["d_in"], dim ** -0.5, 4, 4, qp, kp, bool(causal))
    for got, key in ((dq, "dq"), (dk, "dk"), (dv, "dv")):
        assert np.allclose(got, g[key], atol=1e-12, rtol=0), key


def test_zigzag_positions_balanced():
    G, n = 4, 64
    pos = orc.zigzag_positions(n, G)
    assert sorted(np.concatenate(pos).tolist()) == list(range(n))
    # causal work per rank is equal (the point of zigzag)
    work = [int(sum(orc.causal_allowed(pos[i], pos[j]).sum() for j in range(G)))
            for i in range(G)]
    assert len(set(work)) == 1


def test_bf16_round():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -9, -2.5e-3], np.float32)
    r = orc.bf16_round(x)
    assert r[0] == 1.0 and r[1] == 1.0  # ties to even
    assert r[2] == np.float32(1.0 + 2 ** -7)
    assert abs(r[3] - x[3]) <= abs(x[3]) * 2 ** -8


def test_key_tile_order_matches_reference_golden(golden):
    """local_forward_tiled with a permuted key_tile_order (local_attn.py:212-225),
    causal in global coordinates, 128x128 tiles, against the reference's output."""
    g = golden("lao_order_r256_c640_d64_causal")
    rows, cols, dim, r0, c0, n_total, causal, seed = (int(x) for x in g["meta"])
    qp, kp = np.arange(r0, r0 + rows), np.arange(c0, c0 + cols)
    part = orc.local_forward_tiled(g["q"], g["k"], g["v"], dim ** -0.5, 128, 128, qp, kp,
                                   bool(causal), key_tile_order=list(g["order"]))
    o, lse = part.finalize()
    assert np.max(np.abs(o - g["o"])) < 1e-12
    assert np.max(np.abs(lse - g["lse"])) < 1e-12
    # the order is value-irrelevant to rounding (pkg/tests/test_local_attn.py:145-155)
    o2, lse2 = orc.local_forward_tiled(g["q"], g["k"], g["v"], dim ** -0.5, 128, 128, qp, kp,
                                       bool(causal)).finalize()
    assert np.max(np.abs(o2 - o)) < 1e-13 and np.max(np.abs(lse2 - lse)) < 1e-13
    with pytest.raises(ValueError):
        orc.local_forward_tiled(g["q"], g["k"], g["v"], 0.1, 128, 128, qp, kp, True,
                                key_tile_order=[0, 0, 1, 2, 3])


def test_lao_key_tile_order_must_be_permutation():
    """The product's LAO entry validates the order before touching the device
    (ShapeError, local_attn.py:223-225)."""
    import torch
    from paper_2403_09347_b200 import ShapeError, local_forward
    x = torch.zeros(1, 256, 1, 64)
    with pytest.raises(ShapeError):
        local_forward(x, x, x, key_tile_order=[0, 0])
    with pytest.raises(ShapeError):
        local_forward(x, x, x, key_tile_order=[0, 1, 2])
