"""CPU tests of the host logic: C-ABI exports, hop schedule, ring engine.

The ring engine runs with an oracle-backed kernel provider (tests/oracle_kernels.py)
over (a) the loopback transport (one thread per rank, the reference's threaded
executor) and (b) a real 2-process torch.distributed gloo group.
"""

import os
import re
import subprocess
import sys
import tempfile

import numpy as np
import pytest
import torch

from oracle import burst_oracle as orc
from oracle_kernels import OracleKernels

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "burst_b200.h")


# ---------------------------------------------------------------- C ABI

def test_library_exports_every_header_symbol():
    from paper_2403_09347_b200 import _lib
    declared = set(re.findall(r"BURST_API\s+[\w\s\*]+?\b(burst_\w+)\(", open(HEADER).read()))
    assert declared, "no declarations parsed"
    lib = _lib.load()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.EXPORTED)
    assert lib.burst_version() == 1
    assert lib.burst_workspace_floats(2, 3, 64, 130) == 2 * 3 * 256 * 64


def test_ctypes_structs_match_c_layout():
    from paper_2403_09347_b200 import _lib
    import ctypes
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "burst_b200.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu\n", sizeof(burst_hop), offsetof(burst_hop, softmax_scale),
         offsetof(burst_hop, q_map), sizeof(burst_posmap), sizeof(burst_p2p),
         offsetof(burst_p2p, peer));
  return 0;
}'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "t")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        got = [int(x) for x in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(_lib.Hop), _lib.Hop.softmax_scale.offset, _lib.Hop.q_map.offset,
            ctypes.sizeof(_lib.PosMap), ctypes.sizeof(_lib.P2POp), _lib.P2POp.peer.offset]
    assert got == want


def test_integration_stub():
    """The raw-ctypes binding printed in INTEGRATION.md loads the library and declares
    burst_hop / burst_posmap exactly as the C header lays them out."""
    from paper_2403_09347_b200 import _lib
    import ctypes
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = doc[doc.index("## Reference-side binding"):]
    code = sec[sec.index("```python") + len("```python"):]
    code = code[:code.index("```")]
    lib_path = os.path.join(ROOT, "paper_2403_09347_b200", "libburst_b200.so")
    assert 'ctypes.CDLL("libburst_b200.so")' in code
    ns = {}
    exec(compile(code.replace('"libburst_b200.so"', repr(lib_path)), "INTEGRATION.md", "exec"), ns)
    for mine, ref in ((ns["Hop"], _lib.Hop), (ns["PosMap"], _lib.PosMap)):
        assert ctypes.sizeof(mine) == ctypes.sizeof(ref)
        assert [(f[0], getattr(mine, f[0]).offset) for f in mine._fields_] == \
               [(f[0], getattr(ref, f[0]).offset) for f in ref._fields_]
    assert len(ns["_lib"].burst_lao_fwd.argtypes) == len(_lib._SIGS["burst_lao_fwd"][0])
    assert callable(ns["local_forward_b200"])


def test_errors_map_to_reference_taxonomy():
    from paper_2403_09347_b200 import errors
    assert errors.CODE_TO_ERROR[1] is errors.ShapeError
    assert errors.CODE_TO_ERROR[2] is errors.MaskError
    assert errors.CODE_TO_ERROR[4] is errors.MissingForwardError
    assert issubclass(errors.ShapeError, ValueError)


def test_no_cpu_fallback():
    from paper_2403_09347_b200 import CudaError, burst_attn_func
    q = torch.randn(1, 8, 1, 64, dtype=torch.bfloat16)
    with pytest.raises(CudaError):
        burst_attn_func(q, q, q)


# ---------------------------------------------------------------- schedule

@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("causal,zigzag", [(False, False), (True, False), (True, True)])
def test_hop_plans_cover_exactly_the_visible_pairs(G, causal, zigzag):
    from paper_2403_09347_b200.schedule import plan_hop, shard_map
    n = 8
    N = n * G
    visible = np.zeros((N, N), dtype=int)
    for r in range(G):
        for h in range(G):
            p = plan_hop(r, G, h, n, causal, zigzag)
            assert p.src == (r - h) % G
            if p.skip:
                continue
            qp = np.array(p.q_map.positions(n))[p.q_begin:p.q_begin + p.q_len]
            kp = np.array(p.k_map.positions(n))[p.k_begin:p.k_begin + p.k_len]
            allowed = orc.causal_allowed(qp, kp) if p.causal else np.ones((len(qp), len(kp)), bool)
            for i, a in enumerate(qp):
                for j, b in enumerate(kp):
                    if allowed[i, j]:
                        visible[a, b] += 1
            if not p.causal and causal:
                assert orc.causal_allowed(qp, kp).all(), "unmasked hop must be fully visible"
    want = orc.causal_allowed(np.arange(N), np.arange(N)) if causal else np.ones((N, N), bool)
    assert np.array_equal(visible, want.astype(int))


def test_zigzag_balances_work():
    from paper_2403_09347_b200.schedule import hop_flops, plan_hop
    G, n = 8, 256
    work = [sum(hop_flops(plan_hop(r, G, h, n, True, True), 1, 1, 128)[0] for h in range(G))
            for r in range(G)]
    assert max(work) / min(work) < 1.01
    contiguous = [sum(hop_flops(plan_hop(r, G, h, n, True, False), 1, 1, 128)[0]
                      for h in range(G)) for r in range(G)]
    assert max(contiguous) / min(contiguous) > 4


def test_shard_unshard_roundtrip():
    from paper_2403_09347_b200.schedule import shard, unshard
    x = torch.arange(2 * 48 * 3).reshape(2, 48, 3)
    for zz in (False, True):
        parts = [shard(x, r, 4, zz) for r in range(4)]
        assert torch.equal(unshard(parts, zz), x)


# ---------------------------------------------------------------- engine

def _global_reference(q, k, v, do, causal):
    B, N, H, D = q.shape
    outs = []
    for b in range(B):
        for h in range(H):
            f = lambda t: t[b, :, h].double().numpy()
            dq, dk, dv = orc.backward_dense(f(q), f(k), f(v), f(do), D ** -0.5, causal)
            o, lse = orc.forward_dense(f(q), f(k), f(v), D ** -0.5, causal)
            outs.append((b, h, o, lse, dq, dk, dv))
    return outs


def _check(res, q, k, v, do, causal):
    for b, h, o, lse, dq, dk, dv in _global_reference(q, k, v, do, causal):
        assert np.max(np.abs(res.out[b, :, h].double().numpy() - o)) < 1e-10
        assert np.max(np.abs(res.lse[b, h].double().numpy() - lse)) < 1e-5   # lse is fp32 by contract
        assert np.max(np.abs(res.dq[b, :, h].double().numpy() - dq)) < 1e-5
        assert np.max(np.abs(res.dk[b, :, h].double().numpy() - dk)) < 1e-5
        assert np.max(np.abs(res.dv[b, :, h].double().numpy() - dv)) < 1e-5


@pytest.mark.parametrize("G,causal,zigzag", [(1, False, False), (2, False, False),
                                             (3, False, False), (4, True, False),
                                             (4, True, True), (2, True, True)])
def test_engine_loopback_matches_dense(G, causal, zigzag):
    from paper_2403_09347_b200 import run_ring_pass
    g = torch.Generator().manual_seed(G)
    N = 16 * G
    q, k, v, do = (torch.randn(2, N, 2, 8, generator=g, dtype=torch.float64) for _ in range(4))
    kern = OracleKernels()
    res = run_ring_pass(q, k, v, G, causal=causal, dout=do, zigzag=zigzag, kernels=kern)
    _check(res, q, k, v, do, causal)


def _gloo_worker(rank, world, port, causal, zigzag, out_dir, bwd_payload="kv"):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2403_09347_b200.api import burst_attn_func
    from paper_2403_09347_b200.ring import TorchDistTransport
    from paper_2403_09347_b200.schedule import shard
    from oracle_kernels import OracleKernels as OK
    g = torch.Generator().manual_seed(0)
    N = 24 * world
    q, k, v, do = (torch.randn(1, N, 2, 8, generator=g, dtype=torch.float64) for _ in range(4))
    sh = [shard(t, rank, world, zigzag).requires_grad_(i < 3) for i, t in enumerate((q, k, v, do))]
    o, lse = burst_attn_func(sh[0], sh[1], sh[2], causal=causal, zigzag=zigzag,
                             bwd_payload=bwd_payload, _transport=TorchDistTransport(),
                             _kernels=OK())
    o.backward(sh[3])
    torch.save({"o": o.detach(), "lse": lse, "dq": sh[0].grad, "dk": sh[1].grad,
                "dv": sh[2].grad}, os.path.join(out_dir, f"r{rank}.pt"))
    dist.destroy_process_group()


@pytest.mark.parametrize("causal,zigzag,payload", [(False, False, "kv"), (True, True, "kv"),
                                                   (True, False, "kv"), (True, True, "q")])
def test_engine_gloo_two_processes(causal, zigzag, payload, tmp_path):
    import socket
    import torch.multiprocessing as mp
    from paper_2403_09347_b200.schedule import unshard
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world = 2
    mp.start_processes(_gloo_worker, args=(world, port, causal, zigzag, str(tmp_path), payload),
                       nprocs=world, start_method="spawn", join=True)
    parts = [torch.load(tmp_path / f"r{r}.pt") for r in range(world)]

    class R:
        pass
    res = R()
    res.out = unshard([p["o"] for p in parts], zigzag, 1)
    res.lse = unshard([p["lse"] for p in parts], zigzag, 2)
    res.dq = unshard([p["dq"] for p in parts], zigzag, 1)
    res.dk = unshard([p["dk"] for p in parts], zigzag, 1)
    res.dv = unshard([p["dv"] for p in parts], zigzag, 1)
    g = torch.Generator().manual_seed(0)
    N = 24 * world
    q, k, v, do = (torch.randn(1, N, 2, 8, generator=g, dtype=torch.float64) for _ in range(4))
    _check(res, q, k, v, do, causal)


# ---------------------------------------------------------------- padding (reference pad=True)

@pytest.mark.parametrize("name,zigzag", [("ring_n100_d16_h2_g3_pad_f32", False),
                                         ("ring_n98_d16_h1_g4_causal_pad_f32", False),
                                         ("ring_n98_d16_h1_g4_causal_pad_f32", True)])
def test_engine_padding_matches_reference_golden(golden, name, zigzag):
    """Non-divisible sequence, zero-padded (ring.partition pad=True, ring.py:111-115):
    the engine's ring over oracle kernels must reproduce the reference's outputs."""
    from paper_2403_09347_b200 import run_ring_pass
    g = golden(name)
    seq, dim, heads, gpus, seed, causal, tile, prec = (int(x) for x in g["meta"])
    q, k, v, do, scale = orc.generate_inputs(seq, dim, heads, 1, seed, np.float64)
    to = lambda a: torch.from_numpy(np.ascontiguousarray(a.transpose(1, 0, 2)[None]))
    res = run_ring_pass(to(q), to(k), to(v), gpus, causal=bool(causal), dout=to(do),
                        zigzag=zigzag, kernels=OracleKernels(), pad=True)
    for key, got in (("o", res.out), ("dq", res.dq), ("dk", res.dk), ("dv", res.dv)):
        ref = g[key].transpose(1, 0, 2)[None]
        err = np.max(np.abs(got.numpy() - ref)) / np.max(np.abs(ref))
        assert err < 1e-5, (key, err)
    assert np.max(np.abs(res.lse.numpy() - g["lse"][None])) < 1e-5


def test_padding_required_flag():
    from paper_2403_09347_b200 import ConfigError, run_ring_pass
    x = torch.zeros(1, 10, 1, 8, dtype=torch.float64)
    with pytest.raises(ConfigError):
        run_ring_pass(x, x, x, 4, kernels=OracleKernels())


def test_valid_rows_is_prefix():
    from paper_2403_09347_b200.schedule import shard_map, valid_rows
    for G, n, nv in ((4, 26, 98), (3, 34, 100), (2, 10, 37)):
        for zz in (False, True):
            if zz and n % 2:
                continue
            for r in range(G):
                pos = shard_map(r, G, n, zz).positions(n)
                want = [p < nv for p in pos]
                k = valid_rows(r, G, n, zz, nv)
                assert want == [True] * k + [False] * (n - k)


# ---------------------------------------------------------------- reference payload (f2)

@pytest.mark.parametrize("G,causal,zigzag", [(1, False, False), (2, False, False),
                                             (3, False, False), (4, True, False),
                                             (4, True, True), (3, True, True)])
def test_qtravel_payload_matches_dense(G, causal, zigzag):
    """bwd_payload="q": Q/dO/lse/D travel, K/V/dK/dV pinned (ring.py:65-83, 221-242)."""
    from paper_2403_09347_b200 import run_ring_pass
    g = torch.Generator().manual_seed(10 + G)
    N = 16 * G
    q, k, v, do = (torch.randn(2, N, 2, 8, generator=g, dtype=torch.float64) for _ in range(4))
    res = run_ring_pass(q, k, v, G, causal=causal, dout=do, zigzag=zigzag,
                        kernels=OracleKernels(), bwd_payload="q")
    _check(res, q, k, v, do, causal)


@pytest.mark.parametrize("name,zigzag", [("ring_n100_d16_h2_g3_pad_f32", False),
                                         ("ring_n98_d16_h1_g4_causal_pad_f32", True)])
def test_qtravel_padding_matches_reference_golden(golden, name, zigzag):
    from paper_2403_09347_b200 import run_ring_pass
    g = golden(name)
    seq, dim, heads, gpus, seed, causal, tile, prec = (int(x) for x in g["meta"])
    q, k, v, do, scale = orc.generate_inputs(seq, dim, heads, 1, seed, np.float64)
    to = lambda a: torch.from_numpy(np.ascontiguousarray(a.transpose(1, 0, 2)[None]))
    res = run_ring_pass(to(q), to(k), to(v), gpus, causal=bool(causal), dout=to(do),
                        zigzag=zigzag, kernels=OracleKernels(), pad=True, bwd_payload="q")
    for key, got in (("o", res.out), ("dq", res.dq), ("dk", res.dk), ("dv", res.dv)):
        ref = g[key].transpose(1, 0, 2)[None]
        assert np.max(np.abs(got.numpy() - ref)) / np.max(np.abs(ref)) < 1e-5, key


@pytest.mark.parametrize("causal,zigzag", [(False, False), (True, True)])
def test_qtravel_ledger_counts_fewer_elements(causal, zigzag):
    """The reference payload moves Q + dO (+ lse, D) instead of K + V and fp32 dK + dV:
    ledger element counts from the measured run equal ring_comm_bytes' model."""
    from paper_2403_09347_b200 import run_ring_pass
    G, N, H, D = 4, 64, 2, 8
    g = torch.Generator().manual_seed(3)
    q, k, v, do = (torch.randn(1, N, H, D, generator=g, dtype=torch.float64) for _ in range(4))
    rq = run_ring_pass(q, k, v, G, causal=causal, dout=do, zigzag=zigzag,
                       kernels=OracleKernels(), bwd_payload="q", trace=True)
    n = N // G
    for r, led in enumerate(rq.trace.ledgers):
        from paper_2403_09347_b200.schedule import plan_hop
        parts = sum(1 for h in range(1, G)
                    if not plan_hop((r - h) % G, G, (-h) % G, n, causal, zigzag).skip)
        # Q, dO (n*H*D each), lse + D (H*n each) per rotation; one dQ part per visited block
        assert led.elements_sent_backward == (G - 1) * (2 * n * H * D + 2 * H * n) + parts * n * H * D


# ---------------------------------------------------------------- block-sparse grid masks (f3)

GRID_GOLDENS = [("ring_n64_d16_h2_g4_grid_f64", False, "kv"),
                ("ring_n128_d16_h1_g4_grid_causal_f64", False, "kv"),
                ("ring_n128_d16_h1_g4_grid_causal_f64", True, "kv"),
                ("ring_n128_d16_h1_g4_grid_causal_f64", True, "q")]


@pytest.mark.parametrize("name,zigzag,payload", GRID_GOLDENS)
def test_engine_grid_mask_matches_reference_golden(golden, name, zigzag, payload):
    """BlockGrid masks (masking.py:33-147) through the whole ring engine, against the
    reference's own outputs (tests/golden, made by running the reference)."""
    from paper_2403_09347_b200 import run_ring_pass
    g = golden(name)
    seq, dim, heads, gpus, seed, causal, tile, prec = (int(x) for x in g["meta"])
    q, k, v, do, scale = orc.generate_inputs(seq, dim, heads, 1, seed, np.float64)
    to = lambda a: torch.from_numpy(np.ascontiguousarray(a.transpose(1, 0, 2)[None]))
    spec = {"n_query_blocks": int(g["grid"][0]), "n_key_blocks": int(g["grid"][1]),
            "skip": g["grid_skip"].tolist(), "causal": bool(causal)}
    res = run_ring_pass(to(q), to(k), to(v), gpus, dout=to(do), zigzag=zigzag,
                        kernels=OracleKernels(), mask=spec, bwd_payload=payload)
    # lse is fp32 by contract, so gradients carry its rounding (same bar as
    # test_engine_loopback_matches_dense)
    for key, got, tol in (("o", res.out, 1e-10), ("dq", res.dq, 1e-5), ("dk", res.dk, 1e-5),
                          ("dv", res.dv, 1e-5)):
        ref = g[key].transpose(1, 0, 2)[None]
        assert np.max(np.abs(got.numpy() - ref)) < tol, key
    assert np.max(np.abs(res.lse.numpy() - g["lse"][None])) < 1e-5


def test_grid_mask_validation_and_hop_skip():
    from paper_2403_09347_b200 import MaskError
    from paper_2403_09347_b200.masks import GridMask
    from paper_2403_09347_b200.schedule import plan_hop
    g = GridMask(4, 4, frozenset({(0, 0), (0, 1), (0, 2), (0, 3)})).bind(64)
    with pytest.raises(MaskError):              # query block 0 sees no key
        g.validate(causal=False)
    with pytest.raises(MaskError):
        GridMask(3, 4).bind(64)                  # 3 does not divide 64
    with pytest.raises(MaskError):
        GridMask(2, 2, frozenset({(2, 0)}))      # cell outside the grid
    with pytest.raises(MaskError):               # causal: row 0 only sees key 0
        GridMask(2, 2, frozenset({(0, 0)})).bind(8).validate(causal=True)
    # a hop whose whole rectangle is skipped becomes SKIP (BlockMask.decision)
    g = GridMask(4, 4, frozenset({(1, 3)})).bind(64)
    assert plan_hop(1, 4, 2, 16, False, False, None, g).skip      # queries 16-31 x keys 48-63
    p = plan_hop(1, 4, 1, 16, False, False, None, g)
    assert not p.skip and p.grid is g


def test_grid_mask_from_spec_file(tmp_path):
    from paper_2403_09347_b200.masks import GridMask
    path = tmp_path / "mask.json"
    path.write_text('{"n_query_blocks": 2, "n_key_blocks": 4, "skip": [[1, 0]], "causal": true}')
    g, causal = GridMask.from_spec(str(path))
    assert causal and g.n_query_blocks == 2 and g.skip == frozenset({(1, 0)})
    assert GridMask.from_spec("causal") == (None, True)
    assert GridMask.from_spec(None) == (None, False)


# ---------------------------------------------------------------- bench reference arm

def test_bench_reference_arm_cpu():
    """`bench.py --impl reference` (the driver's reference arm: the reference algorithm on
    the host cores) prints one JSON line with the contract's keys; under torchrun only
    rank 0 prints."""
    import json
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c2",
           "--steps", "1", "--warmup", "0", "--ref-rows", "32"]
    env = dict(os.environ, RANK="0", WORLD_SIZE="1")
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "tokens/s" and d["value"] > 0
    ref_installed = os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "burstsim"))
    assert d["cpu_baseline"]["kind"] == ("reference" if ref_installed else "port")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["extrapolated"] is True
    # same config object as our arm's line (so the driver sees same_config)
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == bench.config_dict(bench.CONFIGS["c2"], 1, "nccl")
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0 and not out.stdout.strip()
