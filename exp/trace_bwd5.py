"""Per-iteration clock64 timeline of LAO-bwd variant 5 (CTA pair), exp/lib_trace.so."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BURST_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), os.environ.get("TRACE_LIB", "lib_trace.so"))
os.environ["BURST_BWD_KERNEL"] = os.environ.get("TRACE_KERNEL", "5")
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
names = {3: "sm:s_full", 4: "sm:p_arrive", 0: "mma:p_full", 11: "mma:S^T+1", 5: "sm:dp_full",
         6: "sm:ds_arrive", 1: "mma:dK", 12: "mma:dQ", 7: "dq:dq_full", 8: "dq:arrive",
         2: "mma:dq_empty", 10: "mma:dOA+1", 9: "dq:issued", 13: "d:ld_done", 14: "d:bar_done",
         15: "d:st_done"}
order = [3, 4, 0, 11, 5, 13, 14, 15, 6, 1, 12, 7, 8, 2, 10, 9]
for c in range(2):
    base = t[c, 3, 0]
    print(f"CTA {c} (0 = leader)")
    print("it " + " ".join(f"{names[e]:>12s}" for e in order))
    for i in range(8, 20):
        print(f"{i:2d} " + " ".join(f"{t[c, e, i] - base:12d}" for e in order))
per = np.diff(t[0, 0, 4:60])
print("leader p_full period median", int(np.median(per)), "cycles")
