"""Kernel-timing experiment (not a test): G=1 forward and backward of a bench
config, CUDA-event timed, for whatever library BURST_LIB points at."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_2403_09347_b200.kernels import CudaKernels  # noqa: E402
from paper_2403_09347_b200.ring import SoloTransport, ring_backward, ring_forward  # noqa: E402

cfg = dict(CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
causal = "causal" in sys.argv[2:]
det = "det" in sys.argv[2:]     # deterministic dQ (ordered reductions)
B, N, H, D = cfg["batch"], cfg["seq"], cfg["heads"], cfg["d"]
q, k, v, do = (torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(4))
kern, tr = CudaKernels(), SoloTransport()
scale = D ** -0.5
f = 4.0 * B * H * N * N * D * (0.5 if causal else 1)
res = {}
for it in range(4):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    o, lse = ring_forward(q, k, v, scale, causal, False, tr, kern)
    e[1].record()
    ring_backward(q, k, v, o, lse, do, scale, causal, False, tr, kern, deterministic=det)
    e[2].record()
    torch.cuda.synchronize()
    res = (e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]))
tag = os.path.basename(os.environ.get("BURST_LIB", "default"))
print(f"{tag:20s} {cfg['seq']} causal={causal} det={det}: fwd {res[0]:8.2f} ms {f / res[0] / 1e9:7.1f} TF/s | "
      f"bwd {res[1]:8.2f} ms {2.5 * f / res[1] / 1e9:7.1f} TF/s", flush=True)
