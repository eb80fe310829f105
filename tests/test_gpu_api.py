"""GPU tests of the public API: autograd through burst_attn_func, error
behaviour of the C ABI (reference taxonomy), rectangular/offset hops."""

import numpy as np
import pytest
import torch

from gpu_utils import make_inputs, max_abs, oracle_ring

pytestmark = pytest.mark.gpu


def test_autograd_single_rank_matches_oracle():
    from paper_2403_09347_b200 import burst_attn_func
    q, k, v, do = make_inputs(2, 384, 3, 128, seed=11)
    qs, ks, vs = (t.clone().requires_grad_(True) for t in (q, k, v))
    o, lse = burst_attn_func(qs, ks, vs, causal=True)
    o.backward(do)
    ro, rlse, dq, dk, dv = oracle_ring(q, k, v, do, 1, True, False)
    assert max_abs(o, ro) < 2e-2 and max_abs(lse, rlse) < 1e-2
    for g, r in ((qs.grad, dq), (ks.grad, dk), (vs.grad, dv)):
        assert max_abs(g, r) < 2e-2


def test_custom_softmax_scale():
    from paper_2403_09347_b200 import run_ring_pass
    q, k, v, do = make_inputs(1, 256, 2, 64, seed=5)
    res = run_ring_pass(q, k, v, 2, softmax_scale=0.3, dout=do)
    ro, rlse, dq, dk, dv = oracle_ring(q, k, v, do, 2, False, False, scale=0.3)
    assert max_abs(res.out, ro) < 2e-2 and max_abs(res.dq, dq) < 2e-2


def test_shape_errors_follow_reference_taxonomy():
    from paper_2403_09347_b200 import ShapeError, UnsupportedError, burst_attn_func
    q = torch.randn(1, 64, 2, 128, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(ShapeError):
        burst_attn_func(q, q[:, :, :1].contiguous(), q)             # head mismatch
    with pytest.raises(ShapeError):
        burst_attn_func(q, q.float(), q)                            # mixed dtypes
    bad = torch.randn(1, 64, 2, 96, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(UnsupportedError):
        burst_attn_func(bad, bad, bad)                              # head_dim 96
    with pytest.raises(ShapeError):
        burst_attn_func(q, q, q, softmax_scale=-1.0)


def test_lao_rectangle_with_global_offsets():
    """One hop over a rectangle in global coordinates (the reference's
    row_offset/col_offset/n_total, local_attn.py:207-212): queries at global
    rows [640, 896) against keys [512, 768), causal -> partial tiles."""
    from oracle import burst_oracle as orc
    from paper_2403_09347_b200.kernels import CudaKernels
    from paper_2403_09347_b200.schedule import HopPlan, PosMap
    q, _, _, _ = make_inputs(1, 256, 2, 128, seed=21)
    _, k, v, _ = make_inputs(1, 256, 2, 128, seed=22)
    plan = HopPlan(0, 0, 0, "diag", 0, 256, 0, 256, True, PosMap(640, 896, 256),
                   PosMap(512, 768, 256))
    o = torch.empty_like(q)
    lse = torch.empty(1, 2, 256, device="cuda")
    CudaKernels().fwd(plan, q, k, v, 128 ** -0.5, None, o, lse, first=True, finalize=True)
    torch.cuda.synchronize()
    f = lambda t: t.float().cpu().numpy().astype(np.float64)
    for h in range(2):
        part = orc.local_forward_tiled(f(q)[0, :, h], f(k)[0, :, h], f(v)[0, :, h],
                                       128 ** -0.5, 128, 128, np.arange(640, 896),
                                       np.arange(512, 768), True)
        ro, rl = part.finalize()
        assert max_abs(o[0, :, h], ro) < 2e-2
        assert max_abs(lse[0, h], rl) < 1e-2


def test_integration_stub_runs_on_gpu():
    """The raw-ctypes binding of INTEGRATION.md (what a maintainer adds to the reference)
    computes one offset causal rectangle like the oracle's local_forward_tiled."""
    import os
    from oracle import burst_oracle as orc
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    doc = open(os.path.join(root, "INTEGRATION.md")).read()
    sec = doc[doc.index("## Reference-side binding"):]
    code = sec[sec.index("```python") + len("```python"):]
    code = code[:code.index("```")]
    lib_path = os.path.join(root, "paper_2403_09347_b200", "libburst_b200.so")
    ns = {}
    exec(compile(code.replace('"libburst_b200.so"', repr(lib_path)), "INTEGRATION.md", "exec"), ns)
    B, H, D, n_q, n_k, r0, c0 = 1, 2, 128, 256, 384, 512, 256
    q, _, _, _ = make_inputs(B, n_q, H, D, seed=21)
    _, k, v, _ = make_inputs(B, n_k, H, D, seed=22)
    scale = D ** -0.5
    out, lse = ns["local_forward_b200"](q, k, v, scale, row_offset=r0, col_offset=c0, causal=True)
    torch.cuda.synchronize()
    for h in range(H):
        f = lambda t: t[0, :, h].float().cpu().numpy().astype(np.float64)
        part = orc.local_forward_tiled(f(q), f(k), f(v), scale, 128, 128,
                                       np.arange(r0, r0 + n_q), np.arange(c0, c0 + n_k), True)
        ro, rl = part.finalize()
        assert np.abs(out[0, :, h].float().cpu().numpy() - ro).max() < 2e-2
        assert np.abs(lse[0, h].cpu().numpy() - rl).max() < 1e-2
