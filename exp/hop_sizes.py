"""Per-hop kernel efficiency vs hop size (the work one rank does per ring hop at N GPUs):
G=1 fwd+bwd of an n x n x 32-head x d128 rectangle, CUDA-event timed, for n = 128K / N."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_09347_b200.kernels import CudaKernels  # noqa: E402
from paper_2403_09347_b200.ring import SoloTransport, ring_backward, ring_forward  # noqa: E402

kern, tr = CudaKernels(), SoloTransport()
H, D = 32, 128
for n in [int(x) for x in (sys.argv[1:] or ["131072", "65536", "32768", "16384", "8192"])]:
    q, k, v, do = (torch.randn(1, n, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(4))
    f = 4.0 * H * n * n * D
    best = None
    for it in range(4 if n >= 65536 else 8):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        o, lse = ring_forward(q, k, v, D ** -0.5, False, False, tr, kern)
        e[1].record()
        ring_backward(q, k, v, o, lse, do, D ** -0.5, False, False, tr, kern)
        e[2].record()
        torch.cuda.synchronize()
        r = (e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]))
        best = r if best is None or sum(r) < sum(best) else best
    print(f"n={n:7d} (N={131072 // n} GPUs per hop): fwd {best[0]:8.2f} ms {f / best[0] / 1e9:7.1f} TF/s | "
          f"bwd {best[1]:8.2f} ms {2.5 * f / best[1] / 1e9:7.1f} TF/s", flush=True)
