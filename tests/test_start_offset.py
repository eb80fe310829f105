"""CPU: start offset of the ring pass (run_ring_pass / burst_attn_func start_offset).

Reference: initial_forward_body (ring.py:137-143) and sim._initial_envelopes
(sim.py:406-419) rotate the initial block assignment -- device i starts with block
(i - start_offset) mod G -- and pkg/tests/test_sim.py:311-321 checks that this only
reorders the merges (values agree to rounding).  The envelope origin check
(sim.py:622-631) maps onto the exchange headers (RingDesyncError).
"""

import numpy as np
import pytest
import torch

from oracle_kernels import OracleKernels


def _pass(q, k, v, do, G, causal, zigzag, payload, offset, mask=None):
    from paper_2403_09347_b200 import run_ring_pass
    return run_ring_pass(q, k, v, G, causal=causal, dout=do, zigzag=zigzag,
                         kernels=OracleKernels(), bwd_payload=payload, start_offset=offset,
                         mask=mask)


def _close(a, b, tol):
    return float(np.max(np.abs(a.double().numpy() - b.double().numpy()))) < tol


@pytest.mark.parametrize("G,causal,zigzag", [(4, False, False), (4, True, True),
                                             (3, True, False), (2, True, True)])
@pytest.mark.parametrize("payload", ["kv", "q"])
def test_start_offset_does_not_change_values(G, causal, zigzag, payload):
    g = torch.Generator().manual_seed(7)
    N = 16 * G
    q, k, v, do = (torch.randn(1, N, 2, 8, generator=g, dtype=torch.float64) for _ in range(4))
    base = _pass(q, k, v, do, G, causal, zigzag, payload, 0)
    for off in (1, 2, G - 1, G + 1, -1):
        rot = _pass(q, k, v, do, G, causal, zigzag, payload, off)
        assert _close(rot.out, base.out, 1e-12), off
        assert _close(rot.lse, base.lse, 1e-5), off     # lse is fp32 by contract
        for name in ("dq", "dk", "dv"):                  # fp32 accumulators, as on the GPU
            assert _close(getattr(rot, name), getattr(base, name), 1e-5), (off, name)


def test_start_offset_with_grid_mask_and_padding():
    spec = {"n_query_blocks": 4, "n_key_blocks": 4, "skip": [[0, 0], [2, 1], [3, 3]]}
    g = torch.Generator().manual_seed(3)
    q, k, v, do = (torch.randn(1, 61, 2, 8, generator=g, dtype=torch.float64) for _ in range(4))
    from paper_2403_09347_b200 import run_ring_pass
    kw = dict(dout=do, kernels=OracleKernels(), pad=True, mask=spec)
    base = run_ring_pass(q, k, v, 4, **kw)
    rot = run_ring_pass(q, k, v, 4, start_offset=3, **kw)
    for name in ("out", "dq", "dk", "dv"):
        assert _close(getattr(rot, name), getattr(base, name), 1e-5), name


def test_start_offset_origin_mismatch_raises_desync():
    """One rank believing in another start offset forwards blocks of the wrong origin:
    the exchange headers catch it (sim.py:622-631 envelope origin check)."""
    from paper_2403_09347_b200 import RingDesyncError
    from paper_2403_09347_b200.ring import ring_forward, run_ranks
    from paper_2403_09347_b200.schedule import shard
    G, N = 4, 64
    g = torch.Generator().manual_seed(1)
    q, k, v = (torch.randn(1, N, 1, 8, generator=g, dtype=torch.float64) for _ in range(3))
    kern = OracleKernels()

    def one(rank, tr):
        sh = [shard(t, rank, G, False) for t in (q, k, v)]
        return ring_forward(*sh, 8 ** -0.5, False, False, tr, kern,
                            offset=2 if rank == 1 else 1)

    with pytest.raises(RingDesyncError):
        run_ranks(G, one)


def test_start_offset_type_checked():
    from paper_2403_09347_b200 import ConfigError, run_ring_pass
    x = torch.zeros(1, 8, 1, 8, dtype=torch.float64)
    with pytest.raises(ConfigError):
        run_ring_pass(x, x, x, 2, kernels=OracleKernels(), start_offset=1.5)
