"""GPU tests of the NCCL ring transport behind the C ABI (burst_ring_*).

On a one-GPU box the communicator has a single rank and every exchange is a
send-to-self (the real NCCL grouped send/recv path of the multi-GPU ring, on a side
stream); the join-stall test shows the watchdog's DeadlockError; the torchrun test
runs the whole ring through NcclTransport on 2, 4 and 8 GPUs and skips itself when
fewer than 2 devices are visible.
"""

import ctypes
import os
import subprocess
import sys
import textwrap

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def _one_rank_ring():
    from paper_2403_09347_b200 import _lib
    lib = _lib.load()
    uid = (ctypes.c_char * 128)()
    _lib.check(lib.burst_ring_unique_id(uid))
    h = ctypes.c_void_p()
    _lib.check(lib.burst_ring_create(uid, 0, 1, torch.cuda.current_device(), 60.0,
                                     ctypes.byref(h)))
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
        _lib.check(lib.burst_ring_wait(h))
        posted, done = ctypes.c_uint64(0), ctypes.c_uint64(0)
        _lib.check(lib.burst_ring_poll(h, ctypes.byref(posted), ctypes.byref(done)))
        assert posted.value == done.value == 2
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


def test_nccl_join_stall_raises_deadlock():
    """Rank 0 of a 2-rank ring whose peer never joins: the non-blocking init is
    abandoned after the timeout with BURST_E_DEADLOCK (DeadlockError) instead of
    hanging (sim.py:290-310)."""
    code = textwrap.dedent("""
        import ctypes, sys, time
        sys.path.insert(0, %r)
        import torch
        from paper_2403_09347_b200 import _lib
        torch.cuda.init()
        lib = _lib.load()
        uid = (ctypes.c_char * 128)()
        _lib.check(lib.burst_ring_unique_id(uid))
        h = ctypes.c_void_p()
        t0 = time.time()
        rc = lib.burst_ring_create(uid, 0, 2, 0, 3.0, ctypes.byref(h))
        print("RC", rc, round(time.time() - t0, 1), lib.burst_last_error().decode())
    """ % ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=240)
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("RC")]
    assert line, r.stdout + r.stderr
    _, rc, secs = line[0].split()[:3]
    assert int(rc) == 7, line[0]                    # BURST_E_DEADLOCK
    assert float(secs) < 60, line[0]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs for a real NCCL ring")
@pytest.mark.parametrize("world", [2, 4, 8])
def test_torchrun_nccl_ring_matches_oracle(world):
    """burst_attn_func through NcclTransport (the bench's N > 1 transport) on `world`
    GPUs: both backward payloads, contiguous and zigzag causal, against the oracle."""
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port",
           str(29600 + world), os.path.join(ROOT, "tests", "nccl_ring_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("RING_OK") == world, r.stdout[-3000:]
