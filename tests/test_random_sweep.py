"""Randomized parity sweep: 128 seeded run_ring_pass configurations (random_cases.py)
that draw every pass option together, checked against the dense fp64 oracle.

CPU (`-m "not gpu"`): the host side -- schedule, zigzag / padding, grid binding,
start offset, both backward payloads, the folds -- driven by the oracle kernels
(tests/oracle_kernels.py) in fp64, to 1e-9, on the first 32 cases.
GPU also runs 24 multi-tile cases (2K-6K tokens, one head).
GPU (`-m gpu`): the same cases through the CUDA kernels: bf16 within 2e-2 max-abs of
the oracle on the same rounded inputs (lse 1e-2), the f32 path within 1e-5 relative
(BASELINE.json north star); deterministic cases also run twice and must agree bit
for bit.
"""

import numpy as np
import pytest
import torch

from random_cases import CASES, CPU_CASES, LARGE_CASES, dense_reference, pass_kwargs


def _id(c):
    return (f"s{c['seed']}-{c['dtype']}-d{c['D']}-g{c['world']}"
            f"{'-causal' if c['causal'] else ''}{'-zz' if c['zigzag'] else ''}"
            f"{'-pad' if c['pad'] else ''}{'-grid' if c['mask'] else ''}-{c['payload']}"
            f"{'-off%d' % c['offset'] if c['offset'] else ''}"
            f"{'-det' if c['deterministic'] else ''}-n{c['N']}")


IDS = [_id(c) for c in CASES]


def _inputs(case, dtype, device):
    g = torch.Generator().manual_seed(case["seed"])
    shape = (case["B"], case["N"], case["H"], case["D"])
    return [torch.randn(*shape, generator=g).to(dtype).to(device) for _ in range(4)]


def _np(t):
    return t.detach().double().cpu().numpy()


def test_cases_cover_every_option():
    """The draw exercises each option at least a few times, already in the CPU subset."""
    for key, want in (("causal", True), ("zigzag", True), ("pad", True),
                      ("deterministic", True), ("payload", "q")):
        assert sum(c[key] == want for c in CPU_CASES) >= 3, key
    assert sum(c["mask"] is not None for c in CPU_CASES) >= 5
    assert sum(c["offset"] > 0 for c in CPU_CASES) >= 3
    assert sum(c["dtype"] == "f32" for c in CPU_CASES) >= 4
    assert {c["world"] for c in CPU_CASES} >= {1, 2, 3, 4, 5, 8}


@pytest.mark.parametrize("case", CPU_CASES, ids=IDS[:len(CPU_CASES)])
def test_host_logic_random_case(case):
    from oracle_kernels import OracleKernels

    from paper_2403_09347_b200 import run_ring_pass
    q, k, v, do = _inputs(case, torch.float64, "cpu")
    kw = pass_kwargs(case)
    kw.pop("deterministic")
    res = run_ring_pass(q, k, v, case["world"], dout=do, kernels=OracleKernels(), **kw)
    o, lse, dq, dk, dv = dense_reference(_np(q), _np(k), _np(v), _np(do), case)
    assert np.max(np.abs(_np(res.out) - o)) < 1e-9
    assert np.max(np.abs(_np(res.lse) - lse)) < 1e-5          # lse is fp32 by contract
    for name, ref in (("dq", dq), ("dk", dk), ("dv", dv)):    # fp32 accumulators
        got = _np(getattr(res, name))
        assert np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-30) < 1e-5, name


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES + LARGE_CASES, ids=IDS + [_id(c) for c in LARGE_CASES])
def test_gpu_random_case(case):
    from gpu_utils import poison_allocator

    from paper_2403_09347_b200 import run_ring_pass
    f32 = case["dtype"] == "f32"
    q, k, v, do = _inputs(case, torch.float32 if f32 else torch.bfloat16, "cuda")
    poison_allocator()
    res = run_ring_pass(q, k, v, case["world"], dout=do, **pass_kwargs(case))
    torch.cuda.synchronize()
    o, lse, dq, dk, dv = dense_reference(_np(q), _np(k), _np(v), _np(do), case)
    for name, got, ref in (("out", res.out, o), ("dq", res.dq, dq), ("dk", res.dk, dk),
                           ("dv", res.dv, dv)):
        err = np.max(np.abs(_np(got) - ref))
        if f32:
            assert err / max(np.max(np.abs(ref)), 1e-30) < 1e-5, name
        else:
            assert err < 2e-2, name
    assert np.max(np.abs(_np(res.lse) - lse)) < (1e-5 if f32 else 1e-2)
    if case["deterministic"]:
        again = run_ring_pass(q, k, v, case["world"], dout=do, **pass_kwargs(case))
        torch.cuda.synchronize()
        for name in ("dq", "dk", "dv"):
            assert torch.equal(getattr(again, name), getattr(res, name)), name
