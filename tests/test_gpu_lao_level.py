"""GPU: the LAO-level entry points (lao.local_forward / local_backward) against the
oracle and the reference's own key_tile_order golden (local_attn.py:207-289).

Tolerances: bf16 <= 2e-2 max-abs against the fp64 oracle on the same bf16-rounded
inputs; f32 <= 1e-5 relative (BASELINE.json north star).
"""

import numpy as np
import pytest
import torch

from gpu_utils import make_inputs, max_abs, rel_err
from oracle import burst_oracle as orc

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2


def _f64(t):
    return t.float().cpu().numpy().astype(np.float64)


def _oracle_fwd(q, k, v, scale, r0, c0, causal, order=None):
    """Per-head oracle (O [n_q, H, D], lse [H, n_q]) of one rectangle, batch 0."""
    qn, kn, vn = _f64(q)[0], _f64(k)[0], _f64(v)[0]
    qp, kp = np.arange(r0, r0 + qn.shape[0]), np.arange(c0, c0 + kn.shape[0])
    o = np.zeros_like(qn)
    lse = np.zeros((qn.shape[1], qn.shape[0]))
    for h in range(qn.shape[1]):
        part = orc.local_forward_tiled(qn[:, h], kn[:, h], vn[:, h], scale, 128, 128, qp, kp,
                                       causal, key_tile_order=order)
        o[:, h], lse[h] = part.finalize()
    return o, lse


def test_key_tile_order_golden_bf16_and_f32(golden):
    from paper_2403_09347_b200 import local_forward
    g = golden("lao_order_r256_c640_d64_causal")
    rows, cols, dim, r0, c0, n_total, causal, seed = (int(x) for x in g["meta"])
    order = [int(x) for x in g["order"]]
    to = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a[None, :, None, :])).to(dt).cuda()
    # f32 path against the reference's own output
    o, lse = local_forward(to(g["q"], torch.float32), to(g["k"], torch.float32),
                           to(g["v"], torch.float32), causal=True, row_offset=r0,
                           col_offset=c0, key_tile_order=order)
    assert rel_err(o[0, :, 0], g["o"]) < 1e-5
    assert rel_err(lse[0, 0], g["lse"]) < 1e-5
    # bf16 path (tcgen05 kernel walks the permuted tiles)
    q, k, v = (to(g[n], torch.bfloat16) for n in ("q", "k", "v"))
    o, lse = local_forward(q, k, v, causal=True, row_offset=r0, col_offset=c0,
                           key_tile_order=order)
    ro, rl = _oracle_fwd(q, k, v, dim ** -0.5, r0, c0, True, order)
    assert max_abs(o[0], ro) < BF16_TOL
    assert max_abs(lse[0], rl) < 1e-3
    assert max_abs(o[0, :, 0], g["o"]) < 5e-2     # bf16 inputs vs the fp64 reference


@pytest.mark.parametrize("causal,r0,c0", [(False, 0, 0), (True, 2048, 0), (True, 1536, 256)])
def test_random_key_tile_order_is_value_irrelevant(causal, r0, c0):
    from paper_2403_09347_b200 import local_forward
    q, _, _, _ = make_inputs(1, 512, 2, 128, seed=5)
    _, k, v, _ = make_inputs(1, 2000, 2, 128, seed=6)      # 16 tiles, the last partial
    order = list(np.random.default_rng(0).permutation(16))
    base_o, base_l = local_forward(q, k, v, causal=causal, row_offset=r0, col_offset=c0)
    o, l = local_forward(q, k, v, causal=causal, row_offset=r0, col_offset=c0,
                         key_tile_order=order)
    torch.cuda.synchronize()
    assert max_abs(o, _f64(base_o)) < BF16_TOL
    assert max_abs(l, _f64(base_l)) < 1e-3
    ro, rl = _oracle_fwd(q, k, v, 128 ** -0.5, r0, c0, causal, order)
    assert max_abs(o[0], ro) < BF16_TOL
    assert max_abs(l[0], rl) < 1e-3


def test_key_tile_order_with_grid_mask():
    from paper_2403_09347_b200 import local_forward
    spec = {"n_query_blocks": 4, "n_key_blocks": 8, "skip": [[0, 1], [1, 3], [2, 7], [3, 0]]}
    q, k, v, _ = make_inputs(1, 1024, 2, 128, seed=9)
    order = list(np.random.default_rng(1).permutation(8))
    base = local_forward(q, k, v, mask=spec)
    perm = local_forward(q, k, v, mask=spec, key_tile_order=order)
    torch.cuda.synchronize()
    assert max_abs(perm[0], _f64(base[0])) < BF16_TOL
    assert max_abs(perm[1], _f64(base[1])) < 1e-3


@pytest.mark.parametrize("causal,r0,c0,nq,nk", [(False, 0, 0, 384, 640), (True, 640, 0, 384, 896),
                                                (True, 512, 128, 300, 700)])
def test_local_backward_matches_oracle(causal, r0, c0, nq, nk):
    from paper_2403_09347_b200 import local_backward, local_forward
    q, _, _, do = make_inputs(1, nq, 2, 128, seed=nq)
    _, k, v, _ = make_inputs(1, nk, 2, 128, seed=nk)
    o, lse = local_forward(q, k, v, causal=causal, row_offset=r0, col_offset=c0)
    dq, dk, dv = local_backward(q, k, v, do, o, lse, causal=causal, row_offset=r0,
                                col_offset=c0)
    torch.cuda.synchronize()
    qn, kn, vn, dn, on = _f64(q)[0], _f64(k)[0], _f64(v)[0], _f64(do)[0], _f64(o)[0]
    ln = lse.double().cpu().numpy()[0]
    qp, kp = np.arange(r0, r0 + nq), np.arange(c0, c0 + nk)
    for h in range(2):
        d_stat = (dn[:, h] * on[:, h]).sum(-1)
        rq, rk, rv = orc.local_backward(qn[:, h], kn[:, h], vn[:, h], dn[:, h], ln[h], d_stat,
                                        128 ** -0.5, 128, 128, qp, kp, causal)
        assert max_abs(dq[0, :, h], rq) < BF16_TOL
        assert max_abs(dk[0, :, h], rk) < BF16_TOL
        assert max_abs(dv[0, :, h], rv) < BF16_TOL
