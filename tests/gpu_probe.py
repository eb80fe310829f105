"""Quick diagnostic on a GPU box: prints per-tensor errors of each kernel path
against a float64 torch reference instead of asserting (one gpurun call gives
the whole picture).  Not collected by pytest."""

import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2403_09347_b200 import run_ring_pass  # noqa: E402


def ref(q, k, v, do, causal):
    q64, k64, v64 = (t.double().requires_grad_() for t in (q, k, v))
    D = q.shape[-1]
    s = torch.einsum("bqhd,bkhd->bhqk", q64, k64) * D ** -0.5
    if causal:
        N = q.shape[1]
        m = torch.ones(N, N, dtype=torch.bool, device=q.device).tril()
        s = s.masked_fill(~m, float("-inf"))
    lse = torch.logsumexp(s, -1)
    p = torch.softmax(s, -1)
    o = torch.einsum("bhqk,bkhd->bqhd", p, v64)
    o.backward(do.double())
    return o.detach(), lse.detach(), q64.grad, k64.grad, v64.grad


def err(a, b):
    return (a.double() - b).abs().max().item()


def case(name, B, N, H, D, world, causal, dtype=torch.bfloat16, zigzag=None):
    g = torch.Generator(device="cpu").manual_seed(0)
    q, k, v, do = (torch.randn(B, N, H, D, generator=g).to(dtype).cuda() for _ in range(4))
    t0 = time.time()
    try:
        res = run_ring_pass(q, k, v, world, causal=causal, dout=do, zigzag=zigzag)
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001
        print(f"{name}: FAILED {type(e).__name__}: {e}", flush=True)
        return
    o, lse, dq, dk, dv = ref(q, k, v, do, causal)
    print(f"{name}: o {err(res.out, o):.2e} lse {err(res.lse, lse):.2e} dq {err(res.dq, dq):.2e} "
          f"dk {err(res.dk, dk):.2e} dv {err(res.dv, dv):.2e} |o| {o.abs().max().item():.2f} "
          f"|dq| {dq.abs().max().item():.2f} ({time.time() - t0:.2f}s)", flush=True)


if __name__ == "__main__":
    print(torch.cuda.get_device_name(), flush=True)
    case("bf16 G1 N256 D128", 1, 256, 2, 128, 1, False)
    case("bf16 G1 N256 D64", 1, 256, 2, 64, 1, False)
    case("bf16 G1 N1000 D128", 2, 1000, 2, 128, 1, False)
    case("bf16 G1 N512 D128 causal", 1, 512, 2, 128, 1, True)
    case("bf16 G2 N512 D128", 1, 512, 2, 128, 2, False)
    case("bf16 G4 N2048 D128 causal zigzag", 1, 2048, 2, 128, 4, True)
    case("f32 G1 N512 D64", 1, 512, 2, 64, 1, False, torch.float32)
    case("f32 G2 N1024 D64 causal", 1, 1024, 2, 64, 2, True, torch.float32, zigzag=False)
