"""Zero-SM ring transport: two processes on ONE GPU exchange
K/V (and dK/dV or dQ contributions) through copy-engine pushes into CUDA-IPC
mailboxes (ring.IpcTransport); results must match the oracle like every other
transport.  Host handshakes over gloo."""

import os
import socket
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, causal, zigzag, payload, out_dir, offset=0):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from gpu_utils import make_inputs
    from paper_2403_09347_b200.api import burst_attn_func
    from paper_2403_09347_b200.ring import IpcTransport
    from paper_2403_09347_b200.schedule import shard
    q, k, v, do = make_inputs(1, 1024, 2, 128, seed=42)
    sh = [shard(t, rank, world, zigzag).requires_grad_(i < 3) for i, t in enumerate((q, k, v, do))]
    tr = IpcTransport()
    for _ in range(2):     # second pass reuses the mailboxes (slot alternation, no regrowth)
        for t in sh[:3]:
            t.grad = None
        o, lse = burst_attn_func(sh[0], sh[1], sh[2], causal=causal, zigzag=zigzag,
                                 bwd_payload=payload, start_offset=offset, _transport=tr)
        o.backward(sh[3])
    torch.cuda.synchronize()
    hu = sorted(tr.host_us)
    cu = sorted(tr.c_us)
    print(f"rank {rank}: host us median {hu[len(hu) // 2]:.1f}, in C {cu[len(cu) // 2]:.1f}, n={len(hu)}",
          flush=True)
    torch.save({"o": o.detach().cpu(), "dq": sh[0].grad.cpu(), "dk": sh[1].grad.cpu(),
                "dv": sh[2].grad.cpu(), "host_us_median": hu[len(hu) // 2]},
               os.path.join(out_dir, f"r{rank}.pt"))
    tr.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("causal,zigzag,payload,offset", [(False, False, "kv", 0),
                                                          (True, True, "kv", 0),
                                                          (True, True, "q", 0),
                                                          (True, True, "kv", 1),
                                                          (False, False, "q", 1)])
def test_ipc_transport_two_processes_one_gpu(causal, zigzag, payload, offset, tmp_path):
    import torch.multiprocessing as mp
    from gpu_utils import make_inputs, max_abs, oracle_ring
    from paper_2403_09347_b200.schedule import unshard
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world = 2
    mp.start_processes(_worker, args=(world, port, causal, zigzag, payload, str(tmp_path), offset),
                       nprocs=world, start_method="spawn", join=True)
    parts = [torch.load(tmp_path / f"r{r}.pt") for r in range(world)]
    q, k, v, do = make_inputs(1, 1024, 2, 128, seed=42)
    o, lse, dq, dk, dv = oracle_ring(q, k, v, do, world, causal, zigzag)
    for key, ref in (("o", o), ("dq", dq), ("dk", dk), ("dv", dv)):
        got = unshard([p[key] for p in parts], zigzag, 1)
        assert max_abs(got, ref) < 2e-2, key
    # an exchange is posted without any host round trip (device-side flags): the
    # host cost is a few driver calls (target < 50 us; loose bound for a busy CI host)
    for p in parts:
        assert p["host_us_median"] < 250.0, p["host_us_median"]
    print("host us per exchange (median per rank):", [round(p["host_us_median"], 1) for p in parts])
