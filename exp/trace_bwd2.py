"""Per-iteration clock64 timeline of the single-CTA LAO-bwd (exp/lib_trace.so)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BURST_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), os.environ.get("TRACE_LIB", "lib_trace.so"))
os.environ["BURST_BWD_KERNEL"] = os.environ.get("TRACE_KERNEL", "1")
import numpy as np, torch
from paper_2403_09347_b200 import _lib
from paper_2403_09347_b200.kernels import CudaKernels
from paper_2403_09347_b200.ring import SoloTransport, ring_backward, ring_forward
N = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
q, k, v, do = (torch.randn(1, N, 32, 128, device="cuda", dtype=torch.bfloat16) for _ in range(4))
kern = CudaKernels()
for _ in range(2):
    o, lse = ring_forward(q, k, v, 128 ** -0.5, False, False, SoloTransport(), kern)
    ring_backward(q, k, v, o, lse, do, 128 ** -0.5, False, False, SoloTransport(), kern)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (32 * 64))()
_lib.load().burst_exp_trace_read(buf)
t = np.array(buf, dtype=np.int64).reshape(2, 16, 64)
names = ["mma:p_full", "mma:ds_full", "mma:dq_empty", "sm:s_full", "sm:p_arrive", "sm:dp_full",
         "sm:ds_arrive", "dq:dq_full", "dq:arrive", "mma:dOb_full", "mma:dOa_next", "mma:Qa_next"]
for c in range(2):
    base = t[c, 3, 0]
    print(f"CTA {c} (pair: 0 = leader): per-iteration timestamps (cycles, relative to sm:s_full[0])")
    print("it " + " ".join(f"{n:>13s}" for n in names))
    for i in range(8, 20):
        print(f"{i:2d} " + " ".join(f"{t[c, e, i] - base:13d}" for e, n in enumerate(names)))
    per = np.diff(t[c, 0, 4:60])
    print("mma:p_full period median", int(np.median(per)), "cycles")
