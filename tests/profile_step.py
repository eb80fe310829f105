"""One warm-up + one measured fwd+bwd step of a bench config, for ncu captures
(`ncu ... python tests/profile_step.py --config c2`).  Not collected by pytest."""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_2403_09347_b200.api import burst_attn_func  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--seq", type=int, default=0)
a = ap.parse_args()
cfg = dict(CONFIGS[a.config])
if a.seq:
    cfg["seq"] = a.seq
B, N, H, D = cfg["batch"], cfg["seq"], cfg["heads"], cfg["d"]
q, k, v, do = (torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(4))
for t in (q, k, v):
    t.requires_grad_(True)
for _ in range(a.steps):
    o, lse = burst_attn_func(q, k, v, causal=cfg["causal"], mask=cfg.get("mask"))
    torch.autograd.grad(o, (q, k, v), do)
torch.cuda.synchronize()
print("done")
