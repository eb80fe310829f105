"""Does an NCCL exchange on the comm stream run while the LAO kernels hold every SM?

One process, a one-rank NCCL ring (burst_ring_*; every exchange is a send-to-self through
NCCL's own kernels), one B200: the backward hop of an 8-GPU C3 ring (16K x 16K x 32
heads) on the compute stream, and the K/V (268 MB) or K/V + fp32 dK/dV (805 MB) payload of
that hop on a high-priority comm stream, posted right after the kernel launch -- the
ring's schedule.  Reports each alone and both together (CUDA events), and the share of
the exchange hidden = 1 - (t_both - t_kernel) / t_exchange.

    python exp/nccl_overlap.py
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_09347_b200 import _lib  # noqa: E402
from paper_2403_09347_b200.kernels import CudaKernels  # noqa: E402
from paper_2403_09347_b200.ring import SoloTransport, ring_backward, ring_forward  # noqa: E402


def main():
    lib = _lib.load()
    uid = (ctypes.c_char * 128)()
    _lib.check(lib.burst_ring_unique_id(uid))
    h = ctypes.c_void_p()
    _lib.check(lib.burst_ring_create(uid, 0, 1, torch.cuda.current_device(), 120.0, ctypes.byref(h)))
    kern, tr = CudaKernels(), SoloTransport()
    n, H, D = 16384, 32, 128
    q, k, v, do = (torch.randn(1, n, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(4))
    o, lse = ring_forward(q, k, v, D ** -0.5, False, False, tr, kern)
    # one hop's LAO backward kernel alone (the per-pass preprocess / finalize are HBM-bound
    # and would meet the copy in HBM, which the per-hop exchange of a ring never does)
    from paper_2403_09347_b200.schedule import FULL, HopPlan, PosMap
    plan = HopPlan(1, 0, 1, FULL, 0, n, 0, n, False, PosMap(0, n, n), PosMap(n, 2 * n, n))
    st = kern.bwd_prepare(o, do, lse)
    dkp, dvp = kern.part(k), kern.part(v)
    hop = lambda: kern.bwd(plan, q, k, v, do, D ** -0.5, st, dkp, dvp, accumulate=False)
    comm = torch.cuda.Stream(priority=-1)
    for label, nbytes in (("fwd payload K/V", 2 * n * H * D * 2),
                          ("bwd payload K/V + fp32 dK/dV", 2 * n * H * D * 2 + 2 * n * H * D * 4)):
        src = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        dst = torch.empty_like(src)
        ops = (_lib.P2POp * 2)()
        ops[0].buf, ops[0].bytes, ops[0].peer, ops[0].is_send = src.data_ptr(), nbytes, 0, 1
        ops[1].buf, ops[1].bytes, ops[1].peer, ops[1].is_send = dst.data_ptr(), nbytes, 0, 0

        def exchange(after=None):
            if after is None:
                comm.wait_stream(torch.cuda.current_stream())
            else:
                comm.wait_event(after)
            _lib.check(lib.burst_ring_sendrecv(h, ops, 2, ctypes.c_void_p(comm.cuda_stream)))

        def once(fn):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            torch.cuda.current_stream().wait_stream(comm)
            b.record()
            torch.cuda.synchronize()
            return a.elapsed_time(b)

        def ce(after=None):   # the "ce" transport's data path: a copy-engine copy (no SM)
            if after is None:
                comm.wait_stream(torch.cuda.current_stream())
            else:
                comm.wait_event(after)
            _lib.check(lib.burst_copy_async(ctypes.c_void_p(dst.data_ptr()),
                                            ctypes.c_void_p(src.data_ptr()), nbytes,
                                            ctypes.c_void_p(comm.cuda_stream)))

        def with_(xfer):
            def fn():
                ev = torch.cuda.Event()
                ev.record()      # the transfer waits only for what preceded the hop's kernel
                hop()
                xfer(ev)         # posted right after the kernel launch (the ring's order)
            return fn

        # interleaved so that clock / power drift hits every variant alike; medians
        fns = {"kernel": hop, "nccl": exchange, "ce": ce, "kernel+nccl": with_(exchange),
               "kernel+ce": with_(ce)}
        for f in fns.values():
            once(f)
        times = {k_: [] for k_ in fns}
        for _ in range(15):
            for name, f in fns.items():
                times[name].append(once(f))
        med = {k_: sorted(v_)[len(v_) // 2] for k_, v_ in times.items()}
        for x in ("nccl", "ce"):
            hid = max(0.0, 1.0 - (med["kernel+" + x] - med["kernel"]) / med[x])
            print(f"{x.upper():4s} {label:30s} {nbytes / 2**20:6.1f} MiB: kernel {med['kernel']:6.2f} ms, "
                  f"transfer {med[x]:5.2f} ms ({nbytes / med[x] / 1e6:6.1f} GB/s), both "
                  f"{med['kernel+' + x]:6.2f} ms -> hidden {hid:.3f}", flush=True)
    lib.burst_ring_destroy(h)


if __name__ == "__main__":
    main()
