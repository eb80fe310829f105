"""Parity at the BASELINE sequence length (128K, configs[2]/[3]) by spot checks:
the CUDA path runs the full 131072-token problem (4 heads x d128, bf16, fwd+bwd);
the fp64 oracle recomputes sampled 128-row blocks of O/lse/dQ against ALL keys and
sampled 128-key blocks of dK/dV against ALL queries (local_forward_tiled /
local_backward with global positions), on the identical
bf16-rounded inputs.  Tolerance: bf16 path <= 2e-2 max-abs (north star)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

N, H, D = 131072, 4, 128
TOL = 2e-2


def _f64(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("causal", [False, True])
def test_128k_spot_checks(causal):
    from oracle import burst_oracle as orc
    from paper_2403_09347_b200.api import burst_attn_func
    g = torch.Generator(device="cuda").manual_seed(7)
    q, k, v, do = (torch.randn(1, N, H, D, device="cuda", generator=g, dtype=torch.bfloat16)
                   for _ in range(4))
    for t in (q, k, v):
        t.requires_grad_(True)
    o, lse = burst_attn_func(q, k, v, causal=causal)
    dq, dk, dv = torch.autograd.grad(o, (q, k, v), do)
    torch.cuda.synchronize()
    scale = D ** -0.5
    pos = np.arange(N)
    rows = [0, 40960, N - 128] if not causal else [128, 65536, N - 128]
    for h in (0, H - 1):
        qh, kh, vh, doh = (_f64(t[0, :, h]) for t in (q, k, v, do))
        oh = _f64(o[0, :, h].detach())
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
