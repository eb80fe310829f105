"""The error boundary on the GPU path: the kernels OR MaskError / NonFiniteError bits into
the pass's device error word; it is read once per pass and raised with the reference's
classes (PartialAttn.finalize, local_attn.py:127-135; linalg._ensure_finite,
linalg.py:253-255)."""

import pytest
import torch

from gpu_utils import make_inputs

pytestmark = pytest.mark.gpu


def _grad(fn, q, k, v, do):
    for t in (q, k, v):
        t.requires_grad_(True)
    o, lse = fn(q, k, v)
    return torch.autograd.grad(o, (q, k, v), do)


@pytest.mark.parametrize("dtype,D", [(torch.bfloat16, 128), (torch.float32, 64)])
def test_inf_in_k_raises_nonfinite_sync(dtype, D):
    from paper_2403_09347_b200 import NonFiniteError, burst_attn_func
    q, k, v, do = make_inputs(1, 512, 2, D, seed=1, dtype=dtype)
    k[0, 100, 1, 5] = float("inf")
    with pytest.raises(NonFiniteError):
        burst_attn_func(q, k, v, check="sync")


def test_nan_in_v_raises_in_ring():
    from paper_2403_09347_b200 import NonFiniteError, run_ring_pass
    q, k, v, do = make_inputs(1, 1024, 2, 128, seed=2)
    v[0, 700, 0, 3] = float("nan")
    with pytest.raises(NonFiniteError):
        run_ring_pass(q, k, v, 2, causal=True, dout=do)


def test_nan_in_dout_raises_in_backward():
    from paper_2403_09347_b200 import NonFiniteError, burst_attn_func
    q, k, v, do = make_inputs(1, 512, 2, 128, seed=3)
    do[0, 7, 1, 0] = float("nan")
    with pytest.raises(NonFiniteError):
        _grad(lambda a, b, c: burst_attn_func(a, b, c, check="sync"), q, k, v, do)


def test_async_check_raises_later():
    """check="async": no host stall at the end of the pass; the error surfaces at the next
    call once the pass has finished, or in check_errors()."""
    from paper_2403_09347_b200 import NonFiniteError, burst_attn_func, check_errors
    q, k, v, do = make_inputs(1, 512, 2, 128, seed=4)
    bad = k.clone()
    bad[0, 0, 0, 0] = float("inf")
    burst_attn_func(q, bad, v, check="async")           # does not raise here
    with pytest.raises(NonFiniteError):
        check_errors()
    check_errors()                                      # consumed: nothing left to raise
    burst_attn_func(q, bad, v, check="async")
    torch.cuda.synchronize()
    with pytest.raises(NonFiniteError):
        burst_attn_func(q, k, v, check="async")         # raised at the next entry
    check_errors()


def test_masked_row_raises_mask_error():
    """A rectangle whose queries all precede its keys (causal): every row is fully masked."""
    from paper_2403_09347_b200 import MaskError
    from paper_2403_09347_b200.kernels import CudaKernels
    from paper_2403_09347_b200.schedule import HopPlan, PosMap
    q, k, v, _ = make_inputs(1, 256, 2, 128, seed=5)
    plan = HopPlan(0, 0, 0, "diag", 0, 256, 0, 256, True, PosMap(0, 256, 256),
                   PosMap(1024, 1280, 256))
    kern = CudaKernels()
    state = kern.fwd_state(q, running=False)
    o = torch.empty_like(q)
    lse = torch.empty(1, 2, 256, device="cuda")
    kern.fwd(plan, q, k, v, 128 ** -0.5, state, o, lse, first=True, finalize=True)
    with pytest.raises(MaskError):
        kern.finish(state, "sync")


def test_clean_pass_raises_nothing():
    from paper_2403_09347_b200 import burst_attn_func, check_errors
    q, k, v, do = make_inputs(1, 1024, 2, 128, seed=6)
    _grad(lambda a, b, c: burst_attn_func(a, b, c, causal=True, check="sync"), q, k, v, do)
    _grad(lambda a, b, c: burst_attn_func(a, b, c, check="async"), q, k, v, do)
    check_errors()
