timeout 200 python exp/cta_life.py 32768 32 det 2>&1 | tail -14
timeout 200 python - <<'PY'
import ctypes, os, sys, numpy as np
os.environ["BURST_LIB"] = "exp/lib_life.so"
sys.path.insert(0, ".")
import torch
from paper_2403_09347_b200 import _lib
from paper_2403_09347_b200.kernels import CudaKernels
from paper_2403_09347_b200.ring import SoloTransport, ring_backward, ring_forward
N, H = 32768, 32
q, k, v, do = (torch.randn(1, N, H, 128, device="cuda", dtype=torch.bfloat16) for _ in range(4))
kern = CudaKernels()
for _ in range(2):
    o, lse = ring_forward(q, k, v, 128 ** -0.5, False, False, SoloTransport(), kern)
    ring_backward(q, k, v, o, lse, do, 128 ** -0.5, False, False, SoloTransport(), kern, deterministic=True)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (65536 * 16))()
_lib.load().burst_exp_life_read(buf)
t = np.array(buf, dtype=np.int64).reshape(65536, 16)[:8192]
e0 = t[:, 0] - t[:, 0].min()
w = (t[:, 8] + t[:, 9]) / 1e3
life = (t[:, 5] - t[:, 0]) / 1e3
for c in list(range(0, 8)) + list(range(140, 156)) + list(range(250, 262)):
    print(c, "start", round(e0[c] / 1e3, 1), "us  life", round(life[c], 1), "us  wait", round(w[c], 1), "us  sm", t[c, 7])
PY
