"""Hidden-communication fractions of the measured loopback ring (trace.py), per
world size and partition: one B200 runs every rank (threads), so kernels of
different ranks share the GPU; the hidden fraction is what the schedule hides."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_09347_b200 import run_ring_pass
from paper_2403_09347_b200.trace import comm_summary
N = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
H = int(sys.argv[2]) if len(sys.argv) > 2 else 16
D = 128
print(f"# exp/trace_ring_summary.py N={N} H={H} D={D} bf16, loopback ring on one B200")
for G, causal in ((2, False), (4, False), (8, False), (4, True), (8, True)):
    for payload in ("kv", "q"):
        q, k, v, do = (torch.randn(1, N, H, D, device="cuda").to(torch.bfloat16) for _ in range(4))
        run_ring_pass(q, k, v, G, causal=causal, dout=do, trace=True, bwd_payload=payload)
        res = run_ring_pass(q, k, v, G, causal=causal, dout=do, trace=True, bwd_payload=payload)
        f, b = comm_summary(res.trace.forward), comm_summary(res.trace.backward)
        print(f"G={G} causal={causal!s:5} payload={payload}: fwd hidden {f['hidden_frac']:.3f} "
              f"stall-hidden {f['stall_hidden_frac']:.3f} exposed {f['exposed_us']:.0f} us "
              f"({f['send_us']:.0f} us sent, {f['compute_us']:.0f} us compute) | bwd hidden "
              f"{b['hidden_frac']:.3f} stall-hidden {b['stall_hidden_frac']:.3f} exposed "
              f"{b['exposed_us']:.0f} us ({b['send_us']:.0f} us sent, {b['compute_us']:.0f} us compute)",
              flush=True)
