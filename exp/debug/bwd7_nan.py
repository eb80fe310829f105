"""Debug: where does the 2-SM backward produce non-finite / wrong values?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import numpy as np, torch
from gpu_utils import make_inputs, oracle_ring
from paper_2403_09347_b200 import run_ring_pass
for N in [int(x) for x in sys.argv[1:]] or [768, 896, 1000, 1024]:
    q, k, v, do = make_inputs(1, N, 2, 128, seed=N)
    res = run_ring_pass(q, k, v, 1, dout=do, check="off")
    torch.cuda.synchronize()
    o, lse, dq, dk, dv = oracle_ring(q, k, v, do, 1, False, False)
    for name, got, ref in (("out", res.out, o), ("dq", res.dq, dq), ("dk", res.dk, dk), ("dv", res.dv, dv)):
        g = got.float().cpu().numpy()
        bad = ~np.isfinite(g)
        err = np.abs(np.where(bad, 0, g) - ref)
        rows_bad = sorted(set(np.nonzero(bad.any(axis=(0, 2, 3)))[0].tolist()))
        rows_err = sorted(set(np.nonzero((err > 2e-2).any(axis=(0, 2, 3)))[0].tolist()))
        print(f"N={N} {name}: nonfinite rows {rows_bad[:8]}{'...' if len(rows_bad) > 8 else ''} ({len(rows_bad)}), "
              f"wrong rows {rows_err[:8]}{'...' if len(rows_err) > 8 else ''} ({len(rows_err)}), max err {err.max():.3e}", flush=True)
