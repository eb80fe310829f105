"""Per-iteration clock64 timeline of LAO-bwd variant 4 (exp/lib_trace.so), CTA 0:
issue/arrive events of every role plus an observer warp's MMA-completion times."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BURST_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), os.environ.get("TRACE_LIB", "lib_trace.so"))
os.environ["BURST_BWD_KERNEL"] = "4"
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
t = np.array(buf, dtype=np.int64).reshape(32, 64)
names = {0: "mma:p_full", 1: "mma:ds_full", 2: "mma:dq_empty", 3: "sm:s_full", 4: "sm:p_arrive",
         5: "sm:dp_full", 6: "sm:ds_arrive", 7: "dq:dq_full", 8: "dq:arrive", 9: "dq:issued",
         10: "mma:do_next", 11: "mma:q_next", 16: "done:S^T", 17: "done:dV", 18: "done:dK+dQ",
         19: "done:dP^T+1", 12: "e:ld_done", 13: "e:exp_done", 14: "e:st_done", 20: "d:ld1_done",
         21: "d:sts_done", 22: "sm1:p_arrive", 23: "sm1:ds_arrive"}
base = t[16, 0]
order = [3, 12, 13, 14, 4, 22, 0, 17, 11, 5, 20, 21, 6, 23, 1, 18, 7, 8, 2, 10, 19, 9]
print("it " + " ".join(f"{names[e]:>11s}" for e in order))
for i in range(8, 24):
    print(f"{i:2d} " + " ".join(f"{t[e, i] - base:11d}" for e in order))
per = np.diff(t[18, 4:60])
print("dK+dQ completion period median", int(np.median(per)), "cycles")
for a, b, lbl in ((16, 4, "S^T done -> P arrive (exp)"), (19, 6, "dP^T done -> dS arrive (WG0)"),
                  (6, 1, "dS arrive(WG0) -> MMA sees ds_full"), (1, 18, "ds_full -> dK+dQ done"),
                  (18, 8, "dK+dQ done -> drain arrive"), (2, 19, "mma dq_empty -> dP^T(i+1) done"),
                  (0, 17, "p_full -> dV done")):
    lag = 1 if b == 6 and a == 19 else 0
    d = t[b, 8 + lag:40 + lag] - t[a, 8:40]
    print(f"{lbl:40s} median {int(np.median(d))}")
