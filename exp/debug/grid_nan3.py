import sys, torch, threading
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from gpu_utils import make_inputs, poison_allocator
from test_gpu_lao import GRID_SPECS
from paper_2403_09347_b200 import run_ring_pass, ring, kernels as K
events = []
def finish(self, state, check, stream=None, where="BurstAttention"):
    s = stream if stream is not None else torch.cuda.current_stream()
    s.synchronize()
    f = int(state.flags.item())
    if f:
        events.append((threading.current_thread().name, type(state).__name__, f))
K.CudaKernels.finish = finish
fails = 0
for it in range(25):
    for payload in ("kv", "q"):
        for (N, world, causal, zigzag, spec) in GRID_SPECS:
            events.clear()
            q, k, v, do = make_inputs(1, N, 2, 128, seed=N + world)
            poison_allocator()
            res = run_ring_pass(q, k, v, world, causal=causal, dout=do, zigzag=zigzag, mask=spec, bwd_payload=payload)
            torch.cuda.synchronize()
            msg = []
            for name in ("out", "lse", "dq", "dk", "dv"):
                t = getattr(res, name).float()
                bad = (~torch.isfinite(t)).nonzero()
                if bad.shape[0]:
                    dim = 2 if name == "lse" else 1
                    rows = sorted(set(bad[:, dim].tolist()))
                    msg.append(f"{name}: {bad.shape[0]} bad, rows {rows[:8]}..{rows[-4:]}")
            if msg or events:
                fails += 1
                print(it, payload, N, world, causal, zigzag, events, "; ".join(msg), flush=True)
print("fails", fails)
