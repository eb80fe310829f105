"""Measured ring timeline and byte ledger in the reference's schema.

The reference simulates a pass on virtual time and exports:
  * ScheduleTrace.to_ndjson (sim.py:186-191): one JSON object per event,
    {"device", "kind", "t_virtual", "round"}, kinds EVENT_KINDS =
    compute_start / compute_end / send_start / send_end / recv_ready (sim.py:159);
  * measure_overlap (sim.py:238-261): per round, |compute ∩ send| / |send|
    averaged over devices (1.0 = transfer fully hidden);
  * CommLedger.to_json (sim.py:118-153): per-device elements sent per pass and
    ring steps.

Here the same records come from the REAL run: CUDA events on each rank's
compute stream (around the hop's LAO kernel) and comm stream (around the hop's
send/recv), resolved after the pass into microseconds since the pass's first
event.  `t_virtual` keeps the reference's key name; its unit is microseconds of
wall time on the device.  On CPU tensors (host-logic tests) the clock is
time.perf_counter.
"""

from __future__ import annotations

import json
import time
from dataclasses import dataclass, field

EVENT_KINDS = ("compute_start", "compute_end", "send_start", "send_end", "recv_ready")


class _Mark:
    __slots__ = ("round", "kind", "event", "t")

    def __init__(self, rnd, kind, event, t):
        self.round, self.kind, self.event, self.t = rnd, kind, event, t


@dataclass
class RingLedger:
    """Per-rank counterpart of CommLedger (sim.py:118-153) for one or more passes:
    elements / bytes this rank sent and the ring steps (exchange slots) taken."""

    elements_sent_forward: int = 0
    elements_sent_backward: int = 0
    bytes_sent_forward: int = 0
    bytes_sent_backward: int = 0
    ring_steps_forward: int = 0
    ring_steps_backward: int = 0

    @property
    def ring_steps(self) -> int:
        return self.ring_steps_forward + self.ring_steps_backward

    def to_json(self) -> dict:
        return {"elements_sent_forward": self.elements_sent_forward,
                "elements_sent_backward": self.elements_sent_backward,
                "bytes_sent_forward": self.bytes_sent_forward,
                "bytes_sent_backward": self.bytes_sent_backward,
                "ring_steps": self.ring_steps,
                "ring_steps_forward": self.ring_steps_forward,
                "ring_steps_backward": self.ring_steps_backward}

    def export(self) -> str:
        return json.dumps(self.to_json(), sort_keys=True)


class PassRecorder:
    """Collects one rank's timeline marks and ledger counts during a pass.

    The hop loops call `mark(round, kind, stream)`; `events()` resolves the
    marks (synchronising the device once) into reference-schema dicts.
    """

    def __init__(self, rank: int = 0):
        self.rank = rank
        self.marks: list[_Mark] = []
        self.ledger = RingLedger()
        self._t0_cpu = None

    def mark(self, rnd: int, kind: str, stream=None) -> None:
        if kind not in EVENT_KINDS:
            raise ValueError(f"unknown event kind {kind!r}")
        if stream is not None:
            import torch
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream)
            self.marks.append(_Mark(rnd, kind, ev, None))
        else:
            self.marks.append(_Mark(rnd, kind, None, time.perf_counter()))

    def count_send(self, phase: str, ops) -> None:
        """Ledger entry for one exchange slot: `ops` = [(kind, tensor, peer[, tag])]."""
        from .ring import SEND
        elems = sum(t.numel() for k, t, *_ in ops if k == SEND)
        nbytes = sum(t.numel() * t.element_size() for k, t, *_ in ops if k == SEND)
        if phase == "forward":
            self.ledger.elements_sent_forward += elems
            self.ledger.bytes_sent_forward += nbytes
            self.ledger.ring_steps_forward += 1
        else:
            self.ledger.elements_sent_backward += elems
            self.ledger.bytes_sent_backward += nbytes
            self.ledger.ring_steps_backward += 1

    def events(self, t0=None) -> list[dict]:
        """Resolve marks into [{"device", "kind", "t_virtual" (us), "round"}]."""
        if not self.marks:
            return []
        if self.marks[0].event is not None:
            self.marks[-1].event.synchronize()
            ref = self.marks[0].event if t0 is None else t0
            out = [(m, ref.elapsed_time(m.event) * 1e3) for m in self.marks]
        else:
            ref = self.marks[0].t if t0 is None else t0
            out = [(m, (m.t - ref) * 1e6) for m in self.marks]
        return [{"device": self.rank, "kind": m.kind, "t_virtual": t, "round": m.round}
                for m, t in out]

    def reference_point(self):
        """The first mark's clock (CUDA event or perf_counter value), for aligning ranks
        that share one device (loopback)."""
        if not self.marks:
            return None
        m = self.marks[0]
        return m.event if m.event is not None else m.t


def merge(recorders, same_clock: bool = True) -> list[dict]:
    """Events of several ranks on one timeline (sorted like ScheduleTrace,
    sim.py:229-230).  Loopback ranks share one device clock, so every rank is
    measured from the earliest rank's first event."""
    recs = [r for r in recorders if r.marks]
    if not recs:
        return []
    t0 = None
    if same_clock:
        firsts = [r.reference_point() for r in recs]
        if recs[0].marks[0].event is not None:
            # pick the earliest CUDA event as the common origin
            t0 = firsts[0]
            for f in firsts[1:]:
                if t0.elapsed_time(f) < 0:
                    t0 = f
        else:
            t0 = min(firsts)
    evs = [e for r in recs for e in r.events(t0)]
    evs.sort(key=lambda e: (e["t_virtual"], e["round"], e["device"], EVENT_KINDS.index(e["kind"])))
    return evs


def to_ndjson(events) -> str:
    """ScheduleTrace.to_ndjson (sim.py:186-191) for measured events."""
    lines = [json.dumps({"device": e["device"], "kind": e["kind"], "t_virtual": e["t_virtual"],
                         "round": e["round"]}, sort_keys=True) for e in events]
    return "\n".join(lines) + ("\n" if lines else "")


def measure_overlap(events) -> dict:
    """measure_overlap (sim.py:238-261) on measured events: per round, the fraction
    of each device's send interval covered by its compute interval, averaged over
    devices; rounds without a send report 0."""
    spans: dict[tuple[int, int], dict[str, float]] = {}
    for e in events:
        spans.setdefault((e["round"], e["device"]), {})[e["kind"]] = e["t_virtual"]
    per_round: dict[int, list[float]] = {}
    for (r, _dev), kinds in sorted(spans.items()):
        if "send_start" not in kinds or "compute_start" not in kinds:
            ratio = 0.0
        else:
            lo = max(kinds["compute_start"], kinds["send_start"])
            hi = min(kinds["compute_end"], kinds["send_end"])
            dur = kinds["send_end"] - kinds["send_start"]
            ratio = max(0.0, hi - lo) / dur if dur > 0 else 0.0
        per_round.setdefault(r, []).append(ratio)
    rounds = {r: sum(v) / len(v) for r, v in per_round.items()}
    mean = sum(rounds.values()) / len(rounds) if rounds else 0.0
    return {"per_round": rounds, "mean": mean}


def comm_summary(events) -> dict:
    """Comm-stream busy time and the share of it hidden under compute, over all
    rounds and devices (north star: >= 90 % of ring communication hidden).

    hidden_frac: the reference's interval overlap (sim.py:238-261) -- the part of
    each send interval covered by the same rank's compute interval of that round.
    stall_hidden_frac: 1 - exposed / send time, where `exposed` is how long the
    compute stream had to wait for an exchange after its kernel of the round had
    finished (recv_ready - compute_end, when positive).  The two agree when every
    rank owns a GPU; when the ranks of a loopback ring share ONE GPU their kernels
    queue behind each other, so a transfer often runs before its own rank's kernel
    has started (not "covered", yet nobody waits for it) -- only the stall measure
    says whether communication cost time there."""
    spans: dict[tuple[int, int], dict[str, float]] = {}
    for e in events:
        spans.setdefault((e["round"], e["device"]), {})[e["kind"]] = e["t_virtual"]
    send_us = hidden_us = exposed_us = compute_us = 0.0
    for kinds in spans.values():
        if "compute_start" in kinds and "compute_end" in kinds:
            compute_us += kinds["compute_end"] - kinds["compute_start"]
        if "send_start" not in kinds:
            continue
        dur = kinds["send_end"] - kinds["send_start"]
        send_us += dur
        if "compute_start" in kinds:
            lo = max(kinds["compute_start"], kinds["send_start"])
            hi = min(kinds["compute_end"], kinds["send_end"])
            hidden_us += max(0.0, hi - lo)
            ready = kinds.get("recv_ready", kinds["send_end"])
            exposed_us += max(0.0, ready - kinds["compute_end"])
        else:
            exposed_us += dur
    return {"send_us": send_us, "hidden_us": hidden_us,
            "hidden_frac": hidden_us / send_us if send_us > 0 else None,
            "exposed_us": exposed_us, "compute_us": compute_us,
            "stall_hidden_frac": max(0.0, 1.0 - exposed_us / send_us) if send_us > 0 else None}


@dataclass
class PassTrace:
    """What `run_ring_pass(..., trace=True)` returns next to the tensors."""
    forward: list = field(default_factory=list)
    backward: list = field(default_factory=list)
    ledgers: list = field(default_factory=list)   # one RingLedger per rank

    def ndjson(self, phase: str = "forward") -> str:
        return to_ndjson(self.forward if phase == "forward" else self.backward)

    def overlap(self, phase: str = "forward") -> dict:
        return measure_overlap(self.forward if phase == "forward" else self.backward)
