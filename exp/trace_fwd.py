"""Per-KV-step clock64 timeline of the LAO forward (exp/lib_trace.so), CTA 0."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BURST_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), os.environ.get("TRACE_LIB", "lib_trace.so"))
import numpy as np, torch
from paper_2403_09347_b200 import _lib
from paper_2403_09347_b200.kernels import CudaKernels
from paper_2403_09347_b200.ring import SoloTransport, ring_forward
N = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
q, k, v = (torch.randn(1, N, 32, 128, device="cuda", dtype=torch.bfloat16) for _ in range(3))
kern = CudaKernels()
for _ in range(3):
    ring_forward(q, k, v, 128 ** -0.5, False, False, SoloTransport(), kern)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (32 * 64))()
_lib.load().burst_exp_trace_read(buf)
t = np.array(buf, dtype=np.int64).reshape(32, 64)
names = {3: "sm0:s_full", 4: "sm0:max", 5: "sm0:p_arr", 11: "sm1:s_full", 12: "sm1:max",
         13: "sm1:p_arr", 0: "mma:V_full", 1: "mma:p0", 2: "mma:p1"}
order = [3, 4, 5, 1, 11, 12, 13, 2, 0]
base = t[3, 0]
print("j  " + " ".join(f"{names[e]:>11s}" for e in order))
for j in range(8, 22):
    print(f"{j:2d} " + " ".join(f"{t[e, j] - base:11d}" for e in order))
print("period (sm0 p_arrive) median", int(np.median(np.diff(t[5, 4:60]))))
for a, b, lbl in ((3, 4, "sm0 ld+max"), (4, 5, "sm0 exp+st"), (5, 1, "sm0 arrive -> mma sees"),
                  (11, 12, "sm1 ld+max"), (12, 13, "sm1 exp+st")):
    print(f"{lbl:26s} median {int(np.median(t[b, 8:40] - t[a, 8:40]))}")
