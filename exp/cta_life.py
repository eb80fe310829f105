"""Where a backward CTA's lifetime goes (experiment, not a test): exp/lib_life.so is the
library built with -DBURST_LIFE (globaltimer at entry, after the setup barrier, when the
first S^T is in TMEM, when the drain issued its last reduction, before and after the
final cluster barrier; slot 7 = SM id).  Reports per-CTA phase medians, the idle gap
between consecutive CTAs on one SM, and how much of SMs x span the main loops cover.

    python -c "from paper_2403_09347_b200 import build as b; b.build(out='exp/lib_life.so', defines=('BURST_LIFE',))"
    python exp/cta_life.py [seq] [heads] [det]
"""
import ctypes
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
os.environ.setdefault("BURST_LIB", os.path.join(HERE, "lib_life.so"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_09347_b200 import _lib  # noqa: E402
from paper_2403_09347_b200.kernels import CudaKernels  # noqa: E402
from paper_2403_09347_b200.ring import SoloTransport, ring_backward, ring_forward  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
H = int(sys.argv[2]) if len(sys.argv) > 2 else 32
DET = "det" in sys.argv[3:]   # deterministic mode: also the turn-wait time per CTA
q, k, v, do = (torch.randn(1, N, H, 128, device="cuda", dtype=torch.bfloat16) for _ in range(4))
kern = CudaKernels()
for _ in range(2):
    o, lse = ring_forward(q, k, v, 128 ** -0.5, False, False, SoloTransport(), kern)
    ring_backward(q, k, v, o, lse, do, 128 ** -0.5, False, False, SoloTransport(), kern,
                  deterministic=DET)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (65536 * 16))()
_lib.load().burst_exp_life_read(buf)
ncta = (N // 128) * H
t = np.array(buf, dtype=np.int64).reshape(65536, 16)[:ncta]
sm = t[:, 7]
e = t[:, :6]
span = e[:, 5].max() - e[:, 0].min()
nsm = len(np.unique(sm))
ph = {"setup (entry -> setup barrier)": e[:, 1] - e[:, 0],
      "first S^T (entry -> S^T_0 in TMEM)": e[:, 2] - e[:, 0],
      "main loop (S^T_0 -> last dQ reduction issued)": e[:, 3] - e[:, 2],
      "tail (last dQ issued -> thread 0 at final barrier)": e[:, 4] - e[:, 3],
      "final cluster barrier": e[:, 5] - e[:, 4],
      "lifetime": e[:, 5] - e[:, 0]}
print(f"N={N} H={H} deterministic={DET}: {ncta} CTAs on {nsm} SMs, kernel span {span / 1e6:.3f} ms")
for name, d in ph.items():
    print(f"  {name:52s} median {np.median(d) / 1e3:8.2f} us  p90 {np.percentile(d, 90) / 1e3:8.2f} us")
gaps = []
for s in np.unique(sm):
    idx = np.where(sm == s)[0]
    idx = idx[np.argsort(e[idx, 0])]
    gaps += list(e[idx[1:], 0] - e[idx[:-1], 5])
gaps = np.array(gaps)
print(f"  idle gap between CTAs on one SM                      median {np.median(gaps) / 1e3:8.2f} us  "
      f"p90 {np.percentile(gaps, 90) / 1e3:8.2f} us  (n={len(gaps)})")
main = (e[:, 3] - e[:, 2]).sum()
busy = (e[:, 5] - e[:, 0]).sum()
print(f"  SM-time: resident {busy / (nsm * span):.3f}, in main loops {main / (nsm * span):.3f} of {nsm} x span")
if DET:
    wa, wb = t[:, 8], t[:, 9]
    print(f"  turn waits: first 32 tiles median {np.median(wa) / 1e3:8.2f} us (p90 {np.percentile(wa, 90) / 1e3:.2f}), "
          f"later tiles median {np.median(wb) / 1e3:8.2f} us (p90 {np.percentile(wb, 90) / 1e3:.2f}) per CTA")
    first = np.argsort(e[:, 0])[:148]
    print(f"  first-wave CTAs: turn waits median {np.median(wa[first] + wb[first]) / 1e3:.2f} us; "
          f"later CTAs {np.median(np.delete(wa + wb, first)) / 1e3:.2f} us")
    even, odd = np.arange(0, ncta, 2), np.arange(1, ncta, 2)
    print(f"  even (pair leader) CTAs wait {np.median(wa[even] + wb[even]) / 1e3:.2f} us, odd {np.median(wa[odd] + wb[odd]) / 1e3:.2f} us")
