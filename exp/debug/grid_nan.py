import sys, torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from gpu_utils import make_inputs, poison_allocator
from paper_2403_09347_b200 import run_ring_pass, ring
spec = {'n_query_blocks': 8, 'n_key_blocks': 8, 'skip': [[3, 1], [5, 2], [7, 0], [6, 6], [2, 0], [4, 3]]}
fails = 0
for it in range(40):
    for payload in ("kv", "q"):
        q, k, v, do = make_inputs(1, 768, 2, 128, seed=770)
        poison_allocator()
        res = run_ring_pass(q, k, v, 2, causal=True, dout=do, zigzag=True, mask=spec, bwd_payload=payload, check="off")
        torch.cuda.synchronize()
        msg = []
        for name in ("out", "lse", "dq", "dk", "dv"):
            t = getattr(res, name).float()
            bad = (~torch.isfinite(t)).nonzero()
            if bad.shape[0]:
                dim = 2 if name == "lse" else 1
                rows = sorted(set(bad[:, dim].tolist()))
                msg.append(f"{name}: {bad.shape[0]} bad, rows {rows[:8]}..{rows[-4:]} heads {sorted(set(bad[:, 2 if dim==1 else 1].tolist()))}")
        if msg:
            fails += 1
            print(it, payload, "; ".join(msg))
print("fails", fails, "of 80")
