"""GPU: the reference's known-answer and property tests (pkg/tests/test_dense.py,
test_local_attn.py) restated for the CUDA path, plus size-independent properties that
also hold at large n: uniform rows, one-hot rows, lse = logsumexp of the scaled scores,
large scores staying finite (the online-softmax rescale), zero upstream gradient,
linearity of dV (and dQ, dK) in dO, and no gradient through masked scores.

Tolerances: bf16 path 2e-2 max-abs against the fp64 oracle on the same rounded inputs;
f32 path 1e-5 relative (BASELINE.json north star).
"""

import numpy as np
import pytest
import torch

from gpu_utils import make_inputs, max_abs, oracle_ring, rel_err

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2


def _ring(q, k, v, do=None, world=1, causal=False, **kw):
    from paper_2403_09347_b200 import run_ring_pass
    res = run_ring_pass(q, k, v, world, causal=causal, dout=do, **kw)
    torch.cuda.synchronize()
    return res


@pytest.mark.parametrize("dtype,D", [(torch.bfloat16, 128), (torch.float32, 64)])
def test_uniform_rows_average_values(dtype, D):
    """q = 0: every score is 0, so each output row is the mean of V and
    lse = log(n) (pkg/tests/test_dense.py:43-51)."""
    n = 1024
    _, k, v, _ = make_inputs(1, n, 2, D, seed=1, dtype=dtype)
    q = torch.zeros_like(k)
    res = _ring(q, k, v, world=2)
    mean = v.double().mean(dim=1, keepdim=True).expand_as(v)
    assert max_abs(res.out, mean.cpu().numpy()) < (BF16_TOL if dtype == torch.bfloat16 else 1e-5)
    assert max_abs(res.lse, np.full((1, 2, n), np.log(n))) < 1e-4


def test_one_hot_rows_select_a_value():
    """Each query equals one key (a permutation) and keys are near-orthogonal with a
    score gap of ~100 after scaling, so every row attends to a single key and
    O_i = v[target_i] (pkg/tests/test_dense.py:53-60)."""
    n, H, D = 512, 2, 128
    g = torch.Generator().manual_seed(3)
    target = torch.randperm(n, generator=g)
    k = torch.randn(1, n, H, D, generator=g) * (40.0 / D ** 0.5)
    q = k[:, target].clone()
    v = torch.randn(1, n, H, D, generator=g)
    q, k, v = (t.to(torch.bfloat16).cuda() for t in (q, k, v))
    res = _ring(q, k, v, world=2)
    assert max_abs(res.out, v[:, target.cuda()].float().cpu().numpy()) < BF16_TOL
    o, lse, *_ = oracle_ring(q, k, v, None, 2, False, False, with_grad=False)
    assert max_abs(res.lse, lse) < 1e-2


@pytest.mark.parametrize("causal", [False, True])
def test_lse_is_logsumexp_of_scaled_scores(causal):
    """lse_i = log sum_j exp(scale q_i.k_j) over visible keys (pkg/tests/test_dense.py),
    in fp64 from the same rounded inputs, for a 2-rank ring."""
    n, H, D = 1024, 2, 128
    q, k, v, _ = make_inputs(1, n, H, D, seed=5)
    res = _ring(q, k, v, world=2, causal=causal, zigzag=causal)
    qd, kd = q.double().cpu()[0], k.double().cpu()[0]
    for h in range(H):
        s = (qd[:, h] @ kd[:, h].T) * D ** -0.5
        if causal:
            s = s.masked_fill(torch.triu(torch.ones(n, n, dtype=torch.bool), 1), float("-inf"))
        ref = torch.logsumexp(s, dim=1).numpy()
        assert max_abs(res.lse[0, h], ref) < 1e-3


@pytest.mark.parametrize("world", [1, 4])
def test_large_scores_stay_finite(world):
    """Scaled scores with a spread of ~+-200 (q, k scaled x 8): the online softmax's lazy
    rescale must keep O, lse and the gradients finite and exact (pkg/tests/test_dense.py
    large-score case)."""
    n, H, D = 2048, 2, 128
    q, k, v, do = make_inputs(1, n, H, D, seed=7)
    q, k = (q.float() * 8).to(torch.bfloat16), (k.float() * 8).to(torch.bfloat16)
    res = _ring(q, k, v, do, world=world)
    for t in (res.out, res.lse, res.dq, res.dk, res.dv):
        assert torch.isfinite(t.float()).all()
    o, lse, dq, dk, dv = oracle_ring(q, k, v, do, world, False, False)
    assert max_abs(res.out, o) < BF16_TOL
    assert max_abs(res.lse, lse) < 5e-2      # |lse| ~ 1e2: fp32 ulps of rounding
    for name, got, ref in (("dq", res.dq, dq), ("dk", res.dk, dk), ("dv", res.dv, dv)):
        assert rel_err(got, ref) < BF16_TOL, name    # gradients scale with |q|, |k|


def test_zero_upstream_gradient_gives_zero_gradients():
    """dO = 0 => dQ = dK = dV = 0 exactly (pkg/tests/test_dense.py backward_zero_upstream)."""
    n, H, D = 1024, 2, 128
    q, k, v, _ = make_inputs(1, n, H, D, seed=9)
    res = _ring(q, k, v, torch.zeros_like(q), world=2, causal=True, zigzag=True)
    for t in (res.dq, res.dk, res.dv):
        assert torch.count_nonzero(t) == 0


@pytest.mark.parametrize("n,world", [(2048, 2), (16384, 4)])
def test_gradients_are_linear_in_upstream(n, world):
    """dQ, dK, dV are linear in dO (pkg/tests/test_dense.py backward_dv_is_linear_map):
    grads(dO1 + dO2) = grads(dO1) + grads(dO2) to bf16 rounding, a size-independent
    check that also runs at a larger n than the oracle would."""
    H, D = 2, 128
    q, k, v, do1 = make_inputs(1, n, H, D, seed=11)
    do2 = make_inputs(1, n, H, D, seed=12)[3]
    do12 = (do1.float() + do2.float()).to(torch.bfloat16)
    r1, r2, r12 = (_ring(q, k, v, d, world=world, causal=True, zigzag=True)
                   for d in (do1, do2, do12))
    for name in ("dq", "dk", "dv"):
        a = getattr(r12, name).float()
        b = getattr(r1, name).float() + getattr(r2, name).float()
        assert float((a - b).abs().max() / a.abs().max()) < BF16_TOL, name


def test_no_gradient_through_masked_scores():
    """A key block no query can see (a block-sparse grid column skipped for every
    query block) receives exactly zero dK and dV, and its values do not change O
    (pkg/tests/test_dense.py gradients_flow_nowhere_through_masked_scores)."""
    n, H, D = 1024, 2, 128
    spec = {"n_query_blocks": 4, "n_key_blocks": 4, "skip": [[0, 2], [1, 2], [2, 2], [3, 2]]}
    q, k, v, do = make_inputs(1, n, H, D, seed=13)
    res = _ring(q, k, v, do, world=2, mask=spec)
    dead = slice(512, 768)
    assert torch.count_nonzero(res.dk[:, dead]) == 0
    assert torch.count_nonzero(res.dv[:, dead]) == 0
    v2 = v.clone()
    v2[:, dead] = 100.0
    res2 = _ring(q, k, v2, do, world=2, mask=spec)
    assert torch.equal(res2.out, res.out)


def test_f32_path_known_answer_hand_case():
    """The reference's hand-checked finalize (pkg/tests/test_local_attn.py:74-79) through
    the kernels: one query, two keys with scores (0, log 2) -> weights (1/3, 2/3)."""
    D = 16
    q = torch.zeros(1, 1, 1, D, dtype=torch.float32)
    k = torch.zeros(1, 2, 1, D, dtype=torch.float32)
    q[..., 0] = 1.0
    k[0, 1, 0, 0] = float(np.log(2.0)) * D ** 0.5      # scaled score = log 2
    v = torch.zeros(1, 2, 1, D, dtype=torch.float32)
    v[0, 0, 0, 0], v[0, 1, 0, 0] = 3.0, 6.0
    from paper_2403_09347_b200 import local_forward
    q1 = torch.zeros(1, 2, 1, D)
    q1[0, :, 0, 0] = 1.0                                    # two identical query rows
    o, lse = local_forward(q1.cuda(), k.cuda(), v.cuda())
    torch.cuda.synchronize()
    assert rel_err(o[0, :, 0, 0], np.array([5.0, 5.0])) < 1e-6     # (3 + 2*6) / 3
    assert max_abs(lse[0, 0], np.full(2, np.log(3.0))) < 1e-6
