"""GPU test of the NCCL ring transport behind the C ABI (burst_ring_*).

Only one GPU is available to the round, so the communicator has a single rank
and every exchange is a send-to-self: this still runs the real NCCL grouped
send/recv path that the multi-GPU ring uses, on a side stream.
"""

import ctypes

import pytest
import torch

pytestmark = pytest.mark.gpu


def _one_rank_ring():
    from paper_2403_09347_b200 import _lib
    lib = _lib.load()
    uid = (ctypes.c_char * 128)()
    _lib.check(lib.burst_ring_unique_id(uid))
    h = ctypes.c_void_p()
    _lib.check(lib.burst_ring_create(uid, 0, 1, torch.cuda.current_device(), ctypes.byref(h)))
    return lib, h


def test_nccl_self_exchange_grouped():
    from paper_2403_09347_b200 import _lib
    lib, h = _one_rank_ring()
    try:
        s = torch.cuda.Stream()
        a = torch.randn(3, 1000, device="cuda")
        b = torch.randn(2, 513, device="cuda", dtype=torch.bfloat16)
        ra, rb = torch.empty_like(a), torch.empty_like(b)
        ops = (_lib.P2POp * 4)()
        for i, (t, send) in enumerate(((a, 1), (b, 1), (ra, 0), (rb, 0))):
            ops[i].buf = t.data_ptr()
            ops[i].bytes = t.numel() * t.element_size()
            ops[i].peer = 0
            ops[i].is_send = send
        s.wait_stream(torch.cuda.current_stream())
        _lib.check(lib.burst_ring_sendrecv(h, ops, 4, ctypes.c_void_p(s.cuda_stream)))
        s.synchronize()
        assert torch.equal(ra, a) and torch.equal(rb, b)
        # single pair entry point
        rc = torch.empty_like(a)
        _lib.check(lib.burst_ring_exchange(h, ctypes.c_void_p(a.data_ptr()),
                                           ctypes.c_void_p(rc.data_ptr()), a.numel() * 4, 0, 0,
                                           ctypes.c_void_p(s.cuda_stream)))
        s.synchronize()
        assert torch.equal(rc, a)
    finally:
        lib.burst_ring_destroy(h)


def test_nccl_rejects_bad_peer():
    from paper_2403_09347_b200 import ShapeError, _lib
    lib, h = _one_rank_ring()
    try:
        ops = (_lib.P2POp * 1)()
        ops[0].buf, ops[0].bytes, ops[0].peer, ops[0].is_send = 0, 4, 3, 1
        with pytest.raises(ShapeError):
            _lib.check(lib.burst_ring_sendrecv(h, ops, 1, ctypes.c_void_p(0)))
    finally:
        lib.burst_ring_destroy(h)
