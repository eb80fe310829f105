"""GPU parity: single-device LAO (G=1) and loopback rings vs the CPU oracle.

Tolerances (BASELINE.json north star): bf16 path <= 2e-2 max-abs against the
reference's fp32 result on identical bf16-rounded inputs; fp32 path <= 1e-5
relative (max|x-ref| / max|ref| per tensor).
"""

import numpy as np
import pytest
import torch

from gpu_utils import make_inputs, max_abs, oracle_ring, poison_allocator, rel_err

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2


def _run(q, k, v, do, world, causal, zigzag=None):
    from paper_2403_09347_b200 import run_ring_pass
    res = run_ring_pass(q, k, v, world, causal=causal, dout=do, zigzag=zigzag)
    torch.cuda.synchronize()
    return res


@pytest.mark.parametrize("N,D", [(256, 128), (512, 128), (384, 64), (1000, 128)])
def test_lao_bf16_single_device(N, D):
    q, k, v, do = make_inputs(1, N, 2, D, seed=N + D)
    res = _run(q, k, v, do, 1, False)
    o, lse, dq, dk, dv = oracle_ring(q, k, v, do, 1, False, False)
    assert max_abs(res.out, o) < BF16_TOL
    assert max_abs(res.lse, lse) < 1e-2
    for got, ref in ((res.dq, dq), (res.dk, dk), (res.dv, dv)):
        assert max_abs(got, ref) < BF16_TOL


@pytest.mark.parametrize("N,D", [(256, 128), (640, 64)])
def test_lao_bf16_causal_single_device(N, D):
    q, k, v, do = make_inputs(2, N, 2, D, seed=7)
    res = _run(q, k, v, do, 1, True)
    o, lse, dq, dk, dv = oracle_ring(q, k, v, do, 1, True, False)
    assert max_abs(res.out, o) < BF16_TOL
    assert max_abs(res.lse, lse) < 1e-2
    for got, ref in ((res.dq, dq), (res.dk, dk), (res.dv, dv)):
        assert max_abs(got, ref) < BF16_TOL


@pytest.mark.parametrize("world,causal,zigzag", [(2, False, False), (4, False, False),
                                                 (2, True, True), (4, True, True),
                                                 (4, True, False), (8, True, True)])
def test_ring_bf16_loopback(world, causal, zigzag):
    N = 256 * world * (2 if zigzag else 1)
    q, k, v, do = make_inputs(1, N, 2, 128, seed=world)
    res = _run(q, k, v, do, world, causal, zigzag)
    o, lse, dq, dk, dv = oracle_ring(q, k, v, do, world, causal, zigzag)
    assert max_abs(res.out, o) < BF16_TOL
    assert max_abs(res.lse, lse) < 1e-2
    for got, ref in ((res.dq, dq), (res.dk, dk), (res.dv, dv)):
        assert max_abs(got, ref) < BF16_TOL


@pytest.mark.parametrize("B,H,N,D,world,causal,zigzag", [
    (2, 3, 1536, 128, 2, True, True),     # batch x heads > 1 through a zigzag ring
    (3, 2, 1024, 64, 4, False, False),    # head_dim 64 bf16 ring
    (2, 1, 2304, 128, 2, False, False),   # shard of 1152 rows: partial last query/key tiles
    (2, 3, 2304, 128, 3, True, True),     # odd ring (G=3), zigzag chunks of 384 rows, 3 key tiles
    (1, 2, 1920, 128, 1, True, False),    # 15 key tiles / 7.5 query blocks: a key-less CTA in the
                                          # last backward pair, a row-less CTA in the last forward pair
    (2, 2, 3840, 128, 5, False, False),   # G=5, 768-row shards: odd cluster counts per hop
])
def test_ring_bf16_batched(B, H, N, D, world, causal, zigzag):
    """Batch and head indexing of every kernel (TMA coordinates, TL workspaces, stats)
    through the ring, including head_dim 64 and shards that are not tile multiples."""
    q, k, v, do = make_inputs(B, N, H, D, seed=B * 100 + H * 10 + world)
    poison_allocator()
    res = _run(q, k, v, do, world, causal, zigzag)
    o, lse, dq, dk, dv = oracle_ring(q, k, v, do, world, causal, zigzag)
    assert max_abs(res.out, o) < BF16_TOL
    assert max_abs(res.lse, lse) < 1e-2
    for name, got, ref in (("dq", res.dq, dq), ("dk", res.dk, dk), ("dv", res.dv, dv)):
        assert max_abs(got, ref) < BF16_TOL, name


@pytest.mark.parametrize("N,D,world,causal", [(512, 64, 1, False), (512, 32, 2, True),
                                              (300, 16, 1, True)])
def test_f32_path_rel_1e5(N, D, world, causal):
    q, k, v, do = make_inputs(1, N, 2, D, seed=3, dtype=torch.float32)
    res = _run(q, k, v, do, world, causal, zigzag=False)
    o, lse, dq, dk, dv = oracle_ring(q, k, v, do, world, causal, False)
    assert rel_err(res.out, o) < 1e-5
    assert max_abs(res.lse, lse) < 1e-4
    for got, ref in ((res.dq, dq), (res.dk, dk), (res.dv, dv)):
        assert rel_err(got, ref) < 1e-5


@pytest.mark.parametrize("N,D,world", [(416, 32, 2), (208, 16, 4)])
def test_f32_zigzag_causal_rel_1e5(N, D, world):
    """Zigzag causal on the f32 path: chunk sizes not a multiple of any tile, partial
    key ranges (K_EARLY_HALF) and query ranges (Q_LATE_HALF); allocator poisoned
    with NaN so an undefined contribution row cannot pass by luck."""
    q, k, v, do = make_inputs(1, N, 2, D, seed=11, dtype=torch.float32)
    poison_allocator()
    res = _run(q, k, v, do, world, True, zigzag=True)
    o, lse, dq, dk, dv = oracle_ring(q, k, v, do, world, True, True)
    assert rel_err(res.out, o) < 1e-5
    for got, ref in ((res.dq, dq), (res.dk, dk), (res.dv, dv)):
        assert rel_err(got, ref) < 1e-5


@pytest.mark.parametrize("N,world", [(800, 2), (1088, 4)])
def test_bf16_zigzag_unaligned_chunks(N, world):
    """bf16 zigzag with chunks of 200 / 136 rows (8- but not 128-aligned): boundary key
    tiles, unaligned Q_LATE_HALF query starts, poisoned allocator."""
    q, k, v, do = make_inputs(1, N, 2, 128, seed=5)
    poison_allocator()
    res = _run(q, k, v, do, world, True, zigzag=True)
    o, lse, dq, dk, dv = oracle_ring(q, k, v, do, world, True, True)
    assert max_abs(res.out, o) < BF16_TOL
    assert max_abs(res.lse, lse) < 1e-2
    for got, ref in ((res.dq, dq), (res.dk, dk), (res.dv, dv)):
        assert max_abs(got, ref) < BF16_TOL


@pytest.mark.parametrize("world,causal,zigzag", [(2, False, False), (4, True, True),
                                                 (4, True, False)])
def test_ring_bf16_reference_payload(world, causal, zigzag):
    """bwd_payload="q" (the reference's Q/dO/lse/D payload, K/V/dK/dV pinned)."""
    from paper_2403_09347_b200 import run_ring_pass
    N = 256 * world * (2 if zigzag else 1)
    q, k, v, do = make_inputs(1, N, 2, 128, seed=20 + world)
    poison_allocator()
    res = run_ring_pass(q, k, v, world, causal=causal, dout=do, zigzag=zigzag, bwd_payload="q")
    torch.cuda.synchronize()
    o, lse, dq, dk, dv = oracle_ring(q, k, v, do, world, causal, zigzag)
    for got, ref in ((res.out, o), (res.dq, dq), (res.dk, dk), (res.dv, dv)):
        assert max_abs(got, ref) < BF16_TOL


def test_f32_reference_payload_rel_1e5():
    from paper_2403_09347_b200 import run_ring_pass
    q, k, v, do = make_inputs(1, 416, 2, 32, seed=12, dtype=torch.float32)
    poison_allocator()
    res = run_ring_pass(q, k, v, 2, causal=True, dout=do, zigzag=True, bwd_payload="q")
    torch.cuda.synchronize()
    o, lse, dq, dk, dv = oracle_ring(q, k, v, do, 2, True, True)
    for got, ref in ((res.dq, dq), (res.dk, dk), (res.dv, dv)):
        assert rel_err(got, ref) < 1e-5


def _grid_oracle(q, k, v, do, world, causal, zigzag, spec):
    """oracle_ring with a block-sparse grid (oracle GridCells = BlockGrid semantics)."""
    from oracle import burst_oracle as orc
    B, N, H, D = q.shape
    grid = orc.GridCells(spec["n_query_blocks"], spec["n_key_blocks"], spec["skip"], N)
    f = lambda t: t.float().cpu().numpy().astype(np.float64)
    qn, kn, vn, dn = f(q), f(k), f(v), f(do)
    out = [np.zeros((B, N, H, D)) for _ in range(4)]
    for b in range(B):
        for h in range(H):
            dq, dk, dv, o, _ = orc.ring_backward(qn[b, :, h], kn[b, :, h], vn[b, :, h],
                                                 dn[b, :, h], D ** -0.5, world, causal, zigzag,
                                                 128, grid)
            for t, x in zip(out, (o, dq, dk, dv)):
                t[b, :, h] = x
    return out


GRID_SPECS = [
    # 128-aligned cells, non-causal, a skipped diagonal cell (own block fully masked)
    (1024, 2, False, False, {"n_query_blocks": 8, "n_key_blocks": 8,
                             "skip": [[0, 0], [1, 5], [2, 2], [3, 7], [6, 1], [7, 7], [4, 4]]}),
    # 96-row cells: cells straddle 128-row tiles (per-element path), causal zigzag
    (768, 2, True, True, {"n_query_blocks": 8, "n_key_blocks": 8,
                          "skip": [[3, 1], [5, 2], [7, 0], [6, 6], [2, 0], [4, 3]]}),
    # own blocks of ranks 0 and 2 fully masked: hop 0 is SKIP (zeroed contribution,
    # forward state starts at the first computed hop)
    (1024, 4, False, False, {"n_query_blocks": 4, "n_key_blocks": 4, "skip": [[0, 0], [2, 2]]}),
    # rectangular grid, causal contiguous, 4 ranks
    (1024, 4, True, False, {"n_query_blocks": 4, "n_key_blocks": 8,
                            "skip": [[1, 0], [2, 3], [3, 1], [3, 6]]}),
]


@pytest.mark.parametrize("N,world,causal,zigzag,spec", GRID_SPECS)
@pytest.mark.parametrize("payload", ["kv", "q"])
def test_bf16_grid_mask(N, world, causal, zigzag, spec, payload):
    """Block-sparse grid masks (BlockGrid, masking.py:33-147) on the bf16 kernels."""
    from paper_2403_09347_b200 import run_ring_pass
    q, k, v, do = make_inputs(1, N, 2, 128, seed=N + world)
    poison_allocator()
    res = run_ring_pass(q, k, v, world, causal=causal, dout=do, zigzag=zigzag,
                        mask=spec, bwd_payload=payload)
    torch.cuda.synchronize()
    o, dq, dk, dv = _grid_oracle(q, k, v, do, world, causal, zigzag, spec)
    for name, got, ref in (("o", res.out, o), ("dq", res.dq, dq), ("dk", res.dk, dk),
                           ("dv", res.dv, dv)):
        assert max_abs(got, ref) < BF16_TOL, name


def test_f32_grid_mask_vs_reference_golden(golden):
    """f32 path with a causal grid mask against the reference's own outputs, 1e-5 rel."""
    from oracle import burst_oracle as orc
    from paper_2403_09347_b200 import run_ring_pass
    g = golden("ring_n256_d32_h1_g2_grid_causal_f32")
    seq, dim, heads, gpus, seed, causal, tile, prec = (int(x) for x in g["meta"])
    qn, kn, vn, dn, scale = orc.generate_inputs(seq, dim, heads, 1, seed, np.float32)
    to = lambda a: torch.from_numpy(np.ascontiguousarray(a.transpose(1, 0, 2)[None])).cuda()
    spec = {"n_query_blocks": int(g["grid"][0]), "n_key_blocks": int(g["grid"][1]),
            "skip": g["grid_skip"].tolist(), "causal": True}
    poison_allocator()
    res = run_ring_pass(to(qn), to(kn), to(vn), gpus, dout=to(dn), mask=spec, zigzag=False)
    torch.cuda.synchronize()
    for key, got in (("o", res.out), ("dq", res.dq), ("dk", res.dk), ("dv", res.dv)):
        assert rel_err(got, g[key].transpose(1, 0, 2)[None]) < 1e-5, key


def test_c1_golden_fp32(golden):
    """BASELINE configs[0] (seq 1024, d 64, 2 heads, G 2, fp32) against the
    reference's own outputs (tests/golden, produced by the reference)."""
    from oracle import burst_oracle as orc
    g = golden("c1_seq1024_d64_h2_g2_f32")
    qn, kn, vn, dn, scale = orc.generate_inputs(1024, 64, 2, 1, 0, np.float32)
    to = lambda a: torch.from_numpy(np.ascontiguousarray(a.transpose(1, 0, 2)[None])).cuda()
    res = _run(to(qn), to(kn), to(vn), to(dn), 2, False)
    for key, got in (("o", res.out), ("dq", res.dq), ("dk", res.dk), ("dv", res.dv)):
        ref = g[key].transpose(1, 0, 2)[None]
        assert rel_err(got, ref) < 1e-5, key
    assert rel_err(res.lse, g["lse"][None]) < 1e-5


@pytest.mark.parametrize("name,zigzag", [("ring_n100_d16_h2_g3_pad_f32", False),
                                         ("ring_n98_d16_h1_g4_causal_pad_f32", False),
                                         ("ring_n98_d16_h1_g4_causal_pad_f32", True)])
def test_f32_padding_vs_reference_golden(golden, name, zigzag):
    """Sequence not divisible by G, zero-padded (reference pad=True): the f32 CUDA
    path against the reference's own outputs, <= 1e-5 relative."""
    from oracle import burst_oracle as orc
    from paper_2403_09347_b200 import run_ring_pass
    g = golden(name)
    seq, dim, heads, gpus, seed, causal, tile, prec = (int(x) for x in g["meta"])
    qn, kn, vn, dn, scale = orc.generate_inputs(seq, dim, heads, 1, seed, np.float32)
    to = lambda a: torch.from_numpy(np.ascontiguousarray(a.transpose(1, 0, 2)[None])).cuda()
    poison_allocator()
    res = run_ring_pass(to(qn), to(kn), to(vn), gpus, causal=bool(causal), dout=to(dn),
                        zigzag=zigzag, pad=True)
    torch.cuda.synchronize()
    for key, got in (("o", res.out), ("dq", res.dq), ("dk", res.dk), ("dv", res.dv)):
        assert rel_err(got, g[key].transpose(1, 0, 2)[None]) < 1e-5, key


@pytest.mark.parametrize("N,world,causal", [(1000, 3, False), (1990, 2, True), (700, 4, False)])
def test_bf16_padding(N, world, causal):
    q, k, v, do = make_inputs(1, N, 2, 128, seed=N)
    from paper_2403_09347_b200 import run_ring_pass
    res = run_ring_pass(q, k, v, world, causal=causal, dout=do, pad=True)
    torch.cuda.synchronize()
    o, lse, dq, dk, dv = oracle_ring(q, k, v, do, 1, causal, False)
    assert max_abs(res.out, o) < BF16_TOL and max_abs(res.lse, lse) < 1e-2
    for got, ref in ((res.dq, dq), (res.dk, dk), (res.dv, dv)):
        assert max_abs(got, ref) < BF16_TOL


@pytest.mark.parametrize("world,payload", [(2, "kv"), (4, "kv"), (8, "kv"), (4, "q"), (8, "q")])
def test_own_block_split_and_folds(world, payload):
    """Rings whose shards are long enough for the own-block split (two 128-aligned query
    halves, the second after hop G-1) and the O(1) contribution folds
    (burst_tl_accumulate), non-causal and causal zigzag, poisoned allocator."""
    for causal, zigzag in ((False, False), (True, True)):
        N = 512 * world * (2 if zigzag else 1)
        q, k, v, do = make_inputs(1, N, 2, 128, seed=40 + world)
        poison_allocator()
        from paper_2403_09347_b200 import run_ring_pass
        res = run_ring_pass(q, k, v, world, causal=causal, dout=do, zigzag=zigzag,
                            bwd_payload=payload)
        torch.cuda.synchronize()
        o, lse, dq, dk, dv = oracle_ring(q, k, v, do, world, causal, zigzag)
        for name, got, ref in (("o", res.out, o), ("dq", res.dq, dq), ("dk", res.dk, dk),
                               ("dv", res.dv, dv)):
            assert max_abs(got, ref) < BF16_TOL, (name, causal)


def test_ring_memory_independent_of_world():
    """O(1) contribution buffers: the peak memory of one rank's backward does not grow
    with the ring size at a fixed local shard (was G-1 held fp32 dK/dV parts)."""
    from paper_2403_09347_b200.api import _default_kernels
    from paper_2403_09347_b200.ring import ring_backward, ring_forward, run_ranks
    from paper_2403_09347_b200.schedule import shard
    n, H = 2048, 4
    kern = _default_kernels()
    per_rank = {}
    for world in (4, 8):
        q, k, v, do = make_inputs(1, n * world, H, 128, seed=world)
        sh = [[shard(t, r, world, False) for r in range(world)] for t in (q, k, v, do)]
        fw = run_ranks(world, lambda rank, tr: ring_forward(sh[0][rank], sh[1][rank], sh[2][rank],
                                                            128 ** -0.5, False, False, tr, kern))
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        run_ranks(world, lambda rank, tr: ring_backward(
            sh[0][rank], sh[1][rank], sh[2][rank], fw[rank][0], fw[rank][1], sh[3][rank],
            128 ** -0.5, False, False, tr, kern))
        torch.cuda.synchronize()
        # loopback ranks share the device: the per-rank figure is the total / world
        per_rank[world] = (torch.cuda.max_memory_allocated() - base) / world
    # held G-1 parts would add 4 fp32 (dK, dV) pairs per rank from G=4 to G=8
    pair = 2 * n * H * 128 * 4
    assert per_rank[8] - per_rank[4] < pair, (per_rank, pair)


def test_unaligned_query_range_reads_only_its_block():
    """A backward hop whose query range starts off the 128-row grid (zigzag
    Q_LATE_HALF) walks the block's 128-row tiles and masks the rows before q_begin;
    the statistics are sized exactly (no slack past the last tile) and come from a
    NaN-poisoned allocator, so a read outside the block or an unmasked row shows up.
    Regression: flaky NonFiniteError in test_bf16_grid_mask[q-768-2-True-True-spec1]."""
    from paper_2403_09347_b200.kernels import CudaKernels
    from paper_2403_09347_b200.schedule import HopPlan, PosMap
    B, n, H, D = 1, 384, 2, 128
    q, k, v, do = make_inputs(B, n, H, D, seed=11)
    scale = D ** -0.5
    kern = CudaKernels()
    full = HopPlan(0, 0, 0, "diag", 0, n, 0, n, False, PosMap(0, n, n), PosMap(0, n, n))
    o = torch.empty_like(q)
    lse = torch.empty(B, H, n, device="cuda")
    kern.fwd(full, q, k, v, scale, kern.fwd_state(q, running=False), o, lse, first=True,
             finalize=True)
    poison_allocator()
    st = kern.bwd_prepare(o, do, lse)
    assert st.stats.numel() == 2 * B * H * 384
    late = HopPlan(0, 0, 0, "diag", 192, n - 192, 0, n, False, PosMap(0, n, n), PosMap(0, n, n))
    dkp, dvp = kern.part(k), kern.part(v)
    kern.bwd(late, q, k, v, do, scale, st, dkp, dvp, accumulate=False)
    dk, dv = torch.empty_like(k), torch.empty_like(v)
    kern.tl_sum([dkp], dk)
    kern.tl_sum([dvp], dv)
    torch.cuda.synchronize()
    # fp64 reference of the same rectangle: rows [192, n) against every key
    f = lambda t: t.double().cpu()[0]
    qd, kd, vd, dod, od = f(q), f(k), f(v), f(do), f(o)
    for h in range(H):
        Q, K, V, dO = qd[192:, h], kd[:, h], vd[:, h], dod[192:, h]
        L = lse.double().cpu()[0, h, 192:]
        P = torch.exp(Q @ K.T * scale - L[:, None])
        Dd = (dO * od[192:, h]).sum(-1)
        dS = P * (dO @ V.T - Dd[:, None])
        ref_dk, ref_dv = scale * dS.T @ Q, P.T @ dO
        assert torch.isfinite(dk[0, :, h]).all()
        assert max_abs(dk[0, :, h], ref_dk.numpy()) < BF16_TOL
        assert max_abs(dv[0, :, h], ref_dv.numpy()) < BF16_TOL


@pytest.mark.parametrize("world,causal,zigzag,payload,offset", [(4, True, True, "kv", 1),
                                                                (4, True, True, "q", 3),
                                                                (3, False, False, "kv", 2),
                                                                (4, True, False, "q", 2)])
def test_ring_start_offset(world, causal, zigzag, payload, offset):
    """start_offset rotates the initial K/V (or query-record) assignment (ring.py:137-143,
    sim.py:406-419): one extra exchange, then the same values as offset 0 to rounding."""
    from paper_2403_09347_b200 import run_ring_pass
    N = 256 * world * (2 if zigzag else 1)
    q, k, v, do = make_inputs(1, N, 2, 128, seed=offset + world)
    poison_allocator()
    res = run_ring_pass(q, k, v, world, causal=causal, dout=do, zigzag=zigzag,
                        bwd_payload=payload, start_offset=offset)
    base = run_ring_pass(q, k, v, world, causal=causal, dout=do, zigzag=zigzag,
                         bwd_payload=payload)
    torch.cuda.synchronize()
    o, lse, dq, dk, dv = oracle_ring(q, k, v, do, world, causal, zigzag)
    assert max_abs(res.out, o) < BF16_TOL
    assert max_abs(res.lse, lse) < 1e-2
    for name, got, ref in (("dq", res.dq, dq), ("dk", res.dk, dk), ("dv", res.dv, dv)):
        assert max_abs(got, ref) < BF16_TOL, name
        assert max_abs(got, getattr(base, name).float().cpu().numpy()) < 1e-2, name
