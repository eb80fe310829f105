"""Parity at the sizes the bench quotes, by spot checks.

The CUDA path runs the whole problem; the fp64 oracle recomputes sampled 128-row
blocks of O/lse/dQ against ALL keys and sampled 128-key blocks of dK/dV against ALL
queries (local_forward_tiled / local_backward with global positions, the reference's
row_offset / col_offset / n_total, local_attn.py:207-248 and 255-289), on the
identical bf16-rounded inputs, in GLOBAL positions (after unshard for rings).
Tolerance: bf16 path <= 2e-2 max-abs (north star).

  * 128K x 4 heads, G=1, causal and not                 (configs[2]/[3] length)
  * C3 exactly: 128K x 32 heads x d128, G=1, heads 0 / 17 / 31
  * C4 exactly: causal, zigzag over G=8 (loopback ring), 16 chunks of 8192, 2 heads
  * C5 shape: 512K x 40 heads x d128, G=1, heads 0 and 39
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

D = 128
TOL = 2e-2


def _f64(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


def _inputs(N, H, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return [torch.randn(1, N, H, D, device="cuda", generator=g, dtype=torch.bfloat16)
            for _ in range(4)]


def spot_check(q, k, v, do, o, lse, dq, dk, dv, heads, rows, causal):
    """Oracle recomputation of sampled query blocks (O, lse, dQ vs every key) and key
    blocks (dK, dV vs every query) of global [1, N, H, D] tensors."""
    from oracle import burst_oracle as orc
    N = q.shape[1]
    scale = D ** -0.5
    pos = np.arange(N)
    for h in heads:
        qh, kh, vh, doh = (_f64(t[0, :, h]) for t in (q, k, v, do))
        oh = _f64(o[0, :, h])
        lseh = lse[0, h].double().cpu().numpy()
        dstat = (doh * oh).sum(axis=1)                       # ring.init_backward D
        for r in rows:
            sl = slice(r, r + 128)
            part = orc.local_forward_tiled(qh[sl], kh, vh, scale, 128, 128, pos[sl], pos, causal)
            o_ref, lse_ref = part.finalize()
            assert np.max(np.abs(oh[sl] - o_ref)) < TOL, ("o", h, r)
            assert np.max(np.abs(lseh[sl] - lse_ref)) < 1e-2, ("lse", h, r)
            dq_ref, _, _ = orc.local_backward(qh[sl], kh, vh, doh[sl], lseh[sl], dstat[sl], scale,
                                              128, 128, pos[sl], pos, causal)
            assert np.max(np.abs(_f64(dq[0, sl, h]) - dq_ref)) < TOL, ("dq", h, r)
            # key block [r, r+128) against every query
            _, dk_ref, dv_ref = orc.local_backward(qh, kh[sl], vh[sl], doh, lseh, dstat, scale,
                                                   128, 128, pos, pos[sl], causal)
            assert np.max(np.abs(_f64(dk[0, sl, h]) - dk_ref)) < TOL, ("dk", h, r)
            assert np.max(np.abs(_f64(dv[0, sl, h]) - dv_ref)) < TOL, ("dv", h, r)


def _attn_g1(N, H, causal, seed):
    from paper_2403_09347_b200.api import burst_attn_func
    q, k, v, do = _inputs(N, H, seed)
    for t in (q, k, v):
        t.requires_grad_(True)
    o, lse = burst_attn_func(q, k, v, causal=causal, check="sync")
    dq, dk, dv = torch.autograd.grad(o, (q, k, v), do)
    torch.cuda.synchronize()
    return q, k, v, do, o, lse, dq, dk, dv


@pytest.mark.parametrize("causal", [False, True])
def test_128k_spot_checks(causal):
    res = _attn_g1(131072, 4, causal, seed=7)
    rows = [0, 40960, 131072 - 128] if not causal else [128, 65536, 131072 - 128]
    spot_check(*res, heads=(0, 3), rows=rows, causal=causal)


def test_c3_32_heads_spot_checks():
    """BASELINE configs[2] at the benchmarked shape: 128K x 32 heads x d128, bf16."""
    res = _attn_g1(131072, 32, False, seed=3)
    spot_check(*res, heads=(0, 17, 31), rows=(8192, 131072 - 128), causal=False)


def test_c4_zigzag_g8_spot_checks():
    """BASELINE configs[3] as specified: causal, zigzag partition over G=8 (16 chunks of
    8192 rows), 128K tokens, through the whole ring (loopback ranks on one GPU)."""
    from paper_2403_09347_b200 import run_ring_pass
    N, H = 131072, 2
    q, k, v, do = _inputs(N, H, seed=11)
    res = run_ring_pass(q, k, v, 8, causal=True, dout=do, zigzag=True)
    torch.cuda.synchronize()
    # rows in early, middle and late chunks: chunk 0 (rank 0), chunk 5 (rank 5),
    # chunk 10 (rank 5's late chunk), the last row block (rank 0's late chunk)
    rows = (0, 5 * 8192 + 4096, 10 * 8192 + 128, N - 128)
    spot_check(q, k, v, do, res.out, res.lse, res.dq, res.dk, res.dv, heads=(0, 1), rows=rows,
               causal=True)


def test_c5_shape_512k_40_heads_spot_checks():
    """BASELINE configs[4] shape (LLaMA-13B attention: 40 heads x d128) at 512K tokens."""
    res = _attn_g1(524288, 40, False, seed=5)
    spot_check(*res, heads=(0, 39), rows=(262144,), causal=False)
