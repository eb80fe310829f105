"""torchrun worker for tests/test_gpu_ring_nccl.py: one rank of a real NCCL ring.

Runs burst_attn_func over NcclTransport (bwd_payload "kv" and "q"; non-causal
contiguous and causal zigzag shards) and compares this rank's outputs and gradients
with the oracle (fp64, identical bf16-rounded inputs), <= 2e-2 max-abs."""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    from gpu_utils import max_abs, oracle_ring
    from paper_2403_09347_b200 import burst_attn_func, check_errors
    from paper_2403_09347_b200.schedule import shard
    for causal, payload in ((False, "kv"), (True, "kv"), (False, "q"), (True, "q")):
        zigzag = causal
        N = 512 * world * (2 if zigzag else 1)
        g = torch.Generator().manual_seed(100 + world)
        q, k, v, do = (torch.randn(1, N, 2, 128, generator=g).to(torch.bfloat16)
                       for _ in range(4))
        sh = [shard(t, rank, world, zigzag).cuda() for t in (q, k, v, do)]
        for t in sh[:3]:
            t.requires_grad_(True)
        o, lse = burst_attn_func(sh[0], sh[1], sh[2], causal=causal, zigzag=zigzag,
                                 bwd_payload=payload, check="sync", deadlock_timeout=120.0)
        dq, dk, dv = torch.autograd.grad(o, sh[:3], sh[3])
        torch.cuda.synchronize()
        ro, rlse, rdq, rdk, rdv = oracle_ring(q, k, v, do, world, causal, zigzag)
        ref = [shard(torch.from_numpy(x), rank, world, zigzag).numpy() for x in (ro, rdq, rdk, rdv)]
        for name, got, want in zip(("o", "dq", "dk", "dv"), (o, dq, dk, dv), ref):
            err = max_abs(got, want)
            assert err < 2e-2, (rank, causal, payload, name, err)
    check_errors()
    dist.barrier()
    print("RING_OK", rank, flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
