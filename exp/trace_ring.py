"""Dump the measured ring timeline of a loopback run (trace.py) for inspection."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_09347_b200 import run_ring_pass
from paper_2403_09347_b200.trace import comm_summary
G = int(sys.argv[1]) if len(sys.argv) > 1 else 2
N, H, D = int(sys.argv[2]) if len(sys.argv) > 2 else 65536, 16, 128
q, k, v, do = (torch.randn(1, N, H, D, device="cuda").to(torch.bfloat16) for _ in range(4))
run_ring_pass(q, k, v, G, dout=do, trace=True)
res = run_ring_pass(q, k, v, G, dout=do, trace=True)
for ph in ("forward", "backward"):
    evs = res.trace.forward if ph == "forward" else res.trace.backward
    print(ph, comm_summary(evs))
    for e in evs:
        print(f"  dev {e['device']} r{e['round']} {e['kind']:14s} {e['t_virtual']:10.1f}")
