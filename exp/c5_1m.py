"""C5 endpoint on one B200: 1M tokens x 40 heads x d128 (LLaMA-13B attention), bf16,
fwd+bwd through burst_attn_func at G=1 -- the whole 1M x 1M score matrix on one GPU,
i.e. 8x the per-GPU work of the 8-GPU weak-scaled endpoint of BASELINE configs[4].

    python exp/c5_1m.py [--seq 1048576] [--steps 1] > profiles/r02_c5_1m.json

Times the steps with CUDA events (one untimed warm-up step first), then checks sampled
128-row blocks of O/lse/dQ against every key and 128-key blocks of dK/dV against every
query with the fp64 oracle (tests/test_gpu_large.spot_check).  Measurement tool, not
product code; the oracle runs only as the checker after the timed region.
"""

import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=1 << 20)
    ap.add_argument("--heads", type=int, default=40)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--no-check", action="store_true")
    a = ap.parse_args()
    from paper_2403_09347_b200.api import burst_attn_func
    N, H, D = a.seq, a.heads, 128
    g = torch.Generator(device="cuda").manual_seed(5)
    q, k, v, do = (torch.randn(1, N, H, D, device="cuda", generator=g, dtype=torch.bfloat16)
                   for _ in range(4))
    for t in (q, k, v):
        t.requires_grad_(True)

    def step():
        o, lse = burst_attn_func(q, k, v, check="async")
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        dq, dk, dv = torch.autograd.grad(o, (q, k, v), do)
        return o, lse, dq, dk, dv, e

    step()                                   # warm-up (allocator, TMA descriptors)
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    fwd_ms, tot_ms = [], []
    for _ in range(a.steps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        o, lse, dq, dk, dv, mid = step()
        e.record()
        torch.cuda.synchronize()
        fwd_ms.append(s.elapsed_time(mid))
        tot_ms.append(s.elapsed_time(e))
    from paper_2403_09347_b200.kernels import check_errors
    check_errors()
    fl_f = 4.0 * N * N * H * D
    fl_b = 2.5 * fl_f
    ms, fm = min(tot_ms), min(fwd_ms)
    out = {"workload": f"C5 endpoint: seq {N} x {H} heads x d{D}, bf16, fwd+bwd, non-causal, "
                       "G=1 (whole score matrix on one B200)",
           "ms_per_step": ms, "fwd_ms": fm, "bwd_ms": ms - fm,
           "tflops": (fl_f + fl_b) / ms / 1e9, "fwd_tflops": fl_f / fm / 1e9,
           "bwd_tflops": fl_b / (ms - fm) / 1e9, "tokens_per_s": N / ms * 1e3,
           "max_memory_gib": torch.cuda.max_memory_allocated() / 2**30,
           "steps": a.steps, "per_gpu_share_at_8_gpus": "1/8 of this step's work"}
    if not a.no_check:
        from test_gpu_large import spot_check
        t0 = time.time()
        spot_check(q, k, v, do, o, lse, dq, dk, dv, heads=(0, H - 1), rows=(N // 2,),
                   causal=False)
        out["parity"] = f"spot checks (heads 0, {H - 1}; rows/keys [{N // 2}, +128)) vs the " \
                        f"fp64 oracle <= 2e-2 max-abs: pass ({time.time() - t0:.0f} s)"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
