"""Failure detection on the ring (CPU, oracle-backed kernels, loopback ranks): the
reference's DeadlockError on a stalled peer (sim.py:290-310, 622-631) and
RingDesyncError on exchange sequence / origin violations (sim.py:570-574)."""

import time

import numpy as np
import pytest
import torch

from oracle_kernels import OracleKernels


def _inputs(G, N_per=16, seed=0):
    g = torch.Generator().manual_seed(seed)
    return [torch.randn(1, N_per * G, 2, 8, generator=g, dtype=torch.float64) for _ in range(4)]


def test_stalled_rank_raises_deadlock_within_timeout():
    from paper_2403_09347_b200 import DeadlockError
    from paper_2403_09347_b200.ring import ring_forward, run_ranks
    from paper_2403_09347_b200.schedule import shard
    G = 3
    q, k, v, _ = _inputs(G)
    sh = [[shard(t, r, G, False) for r in range(G)] for t in (q, k, v)]
    kern = OracleKernels()

    def one(rank, transport):
        if rank == 2:
            time.sleep(3.0)              # a peer that stops making progress
        return ring_forward(sh[0][rank], sh[1][rank], sh[2][rank], 8 ** -0.5, False, False,
                            transport, kern)

    t0 = time.time()
    with pytest.raises(DeadlockError):
        run_ranks(G, one, deadlock_timeout=0.5)
    assert time.time() - t0 < 20


def test_run_ring_pass_deadlock_timeout_parameter():
    """run_ring_pass(deadlock_timeout=...) bounds a healthy pass too (no false alarm)."""
    from paper_2403_09347_b200 import run_ring_pass
    q, k, v, do = _inputs(2)
    res = run_ring_pass(q, k, v, 2, dout=do, kernels=OracleKernels(), deadlock_timeout=30.0)
    assert res.dq is not None


def test_desynchronised_pass_raises_ring_desync():
    """A rank whose pass counter disagrees with its peers' (it ran an extra pass, or
    skipped one) is caught by the exchange headers at the end of the pass."""
    from paper_2403_09347_b200 import RingDesyncError
    from paper_2403_09347_b200.ring import ring_forward, run_ranks
    from paper_2403_09347_b200.schedule import shard
    G = 2
    q, k, v, _ = _inputs(G)
    sh = [[shard(t, r, G, False) for r in range(G)] for t in (q, k, v)]
    kern = OracleKernels()

    def one(rank, transport):
        if rank == 1:
            transport.next_pass()        # rank 1 believes this is its second pass
        return ring_forward(sh[0][rank], sh[1][rank], sh[2][rank], 8 ** -0.5, False, False,
                            transport, kern)

    with pytest.raises(RingDesyncError):
        run_ranks(G, one, deadlock_timeout=10.0)


def test_slot_log_catches_wrong_origin_and_slot():
    from paper_2403_09347_b200 import RingDesyncError
    from paper_2403_09347_b200.ring import SlotLog, _rotating, backward_slots

    class T:
        rank, world, pass_seq = 2, 4, 0

        def next_pass(self):
            self.pass_seq += 1
            return self.pass_seq

    log = SlotLog(T(), torch.device("cpu"), backward_slots(4), _rotating(4))
    good = log.expected.copy()
    log._check(torch.from_numpy(good))                      # consistent: no error
    assert [int(x) for x in good[:, 1]] == [0, 1, 2, 3, 4]  # K/V slots 0-2, homecomings 2-4
    assert list(good[0]) == [1, 0, 1, 1] and good[3][3] == -1
    bad = good.copy()
    bad[1, 3] = 3                                           # a block from the wrong origin
    with pytest.raises(RingDesyncError):
        log._check(torch.from_numpy(bad))
    bad = good.copy()
    bad[2, 1] = 7                                           # an out-of-sequence exchange
    with pytest.raises(RingDesyncError):
        log._check(torch.from_numpy(bad))


def test_exchange_headers_travel_in_every_slot():
    """Every exchange slot of both passes moves one header to rank+1, so the headers a
    rank receives are exactly its predecessor's schedule."""
    from paper_2403_09347_b200.ring import LoopbackHub, ring_backward, ring_forward, run_ranks
    from paper_2403_09347_b200.schedule import shard
    G = 4
    q, k, v, do = _inputs(G)
    sh = [[shard(t, r, G, True) for r in range(G)] for t in (q, k, v, do)]
    kern = OracleKernels()
    seen = {}

    def one(rank, transport):
        orig = transport.sendrecv

        def spy(ops, stream):
            hdr = [t for kind, t, peer, *_ in ops if t.dtype == torch.int32]
            seen.setdefault(rank, []).append(len(hdr))
            return orig(ops, stream)
        transport.sendrecv = spy
        o, lse = ring_forward(sh[0][rank], sh[1][rank], sh[2][rank], 8 ** -0.5, True, True,
                              transport, kern)
        return ring_backward(sh[0][rank], sh[1][rank], sh[2][rank], o, lse, sh[3][rank],
                             8 ** -0.5, True, True, transport, kern)

    run_ranks(G, one)
    # forward: G-1 slots; backward: G-1 K/V slots + homecomings at h = 2..G-1 and G
    for r in range(G):
        assert seen[r] == [2] * ((G - 1) + (G + 1))
