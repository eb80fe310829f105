#!/usr/bin/env python
"""BurstAttention forward+backward benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3|c2|c4|c5_512k]
                    [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...       (N > 1, one rank per GPU)

One step = forward + backward of attention over the whole global sequence,
each rank holding N/G rows (contiguous shards; zigzag shards when causal) and
the K/V (+ dK/dV) ring running over NCCL.  Prints ONE JSON line on rank 0.

  value   whole-job tokens/s, device-timed (CUDA events, max over ranks),
          inputs resident in HBM (every input tensor is 1 GiB at c3 >> 126 MB L2)
  e2e     the same through burst_attn_func with pinned HOST buffers: H2D of
          q/k/v/dO and D2H of out/dq/dk/dv inside the timed region, pipelined
          across steps like a training loop (two copy streams)
  roofline  live per-launch timing of the dominant kernel (LAO backward) on its
          stream; algorithmic FLOPs = 10*B*H*visible(q,k)*d per launch
  cpu_baseline  the reference algorithm (oracle port, numpy/OpenBLAS) on a
          bounded sample of the same workload on this host, extrapolated
--impl reference times only that CPU path (rank 0), same metric/unit.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("attn fwd+bwd TFLOP/s/GPU & tokens/s at 128K seq, 1/2/4/8 B200; % of TC peak")
CONFIGS = {
    "c3": dict(workload="LLaMA-7B-shaped attention, seq 128K, 32 heads x d128, bf16, fwd+bwd, "
                        "non-causal, ring over the N GPUs (BASELINE configs[2])",
               seq=131072, heads=32, d=128, batch=1, causal=False),
    "c2": dict(workload="single-GPU LAO, seq 32K, 32 heads x d128, bf16, non-causal "
                        "(BASELINE configs[1])", seq=32768, heads=32, d=128, batch=1, causal=False),
    "c4": dict(workload="causal LLaMA-7B-shaped attention, seq 128K, zigzag partition, bf16, "
                        "fwd+bwd (BASELINE configs[3])", seq=131072, heads=32, d=128, batch=1,
               causal=True),
    "c3_sparse": dict(workload="C3 shape with a block-sparse grid mask: 32x32 cells of 4096 "
                               "positions, checkerboard of skipped cells (50% of the score matrix), "
                               "non-causal (reference BlockGrid, masking.py:33-147)",
                      seq=131072, heads=32, d=128, batch=1, causal=False,
                      mask={"n_query_blocks": 32, "n_key_blocks": 32,
                            "skip": [[a, b] for a in range(32) for b in range(32) if (a + b) % 2]}),
    "c5_512k": dict(workload="LLaMA-13B-shaped attention, 40 heads x d128, seq 512K, bf16, "
                             "fwd+bwd (BASELINE configs[4])", seq=524288, heads=40, d=128,
                    batch=1, causal=False),
}


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:  # noqa: BLE001
        return {}


# ----------------------------------------------------------------- clocks

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.path = tempfile.mktemp(suffix=".csv")
        self.proc = None
        self.gpu = gpu_index

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)], stdout=open(self.path, "w"),
                stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None
        # nvidia-smi needs ~0.5-1 s before its first sample: wait for it so short timed
        # regions (C2: ~0.3 s) are sampled; rows before the region are dropped below
        t0 = time.time()
        while self.proc is not None and time.time() - t0 < 5.0:
            if self._lines():
                break
            time.sleep(0.05)
        self.skip = len(self._lines())
        return self

    def _lines(self):
        try:
            return [ln for ln in open(self.path) if ln.strip()]
        except Exception:  # noqa: BLE001
            return []

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        rows = []
        for line in self._lines()[getattr(self, "skip", 0):]:
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9 and f[1].replace(".", "").isdigit():
                rows.append(f)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][2]),
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit())}


# ----------------------------------------------------------------- CPU reference

REF_PATH = os.path.join(ROOT, "baseline", "_ref")


def _stock_reference():
    """The unmodified reference package (pip-installed into baseline/_ref), or None."""
    if os.path.isdir(REF_PATH) and REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    try:
        from burstsim import local_attn, masking   # noqa: F401
        from burstsim.linalg import Matrix, Vector  # noqa: F401
        return local_attn
    except Exception:  # noqa: BLE001
        return None


def cpu_reference_sample(cfg, world: int, rows: int = 512):
    """The reference's LAO kernels on `rows` query rows x ALL keys of one head, fwd+bwd:
    the stock `burstsim.local_attn.local_forward_tiled` + `PartialAttn.finalize` +
    `local_backward` (local_attn.py:207-289) from baseline/_ref when installed (kind
    "reference"), else the oracle port of the same tiled algorithm (kind "port").
    128x128 tiles (the reference's own default for d=128 fp32 is 2x2, TileSpec.
    for_partition local_attn.py:44-58, which would take hours), fp32 (the reference's
    "single" precision), global positions via row_offset / n_total.
    Returns (seconds, extrapolation factor to the whole global step, kind)."""
    import numpy as np
    N, d = cfg["seq"], cfg["d"]
    rng = np.random.default_rng(0)
    q = rng.standard_normal((rows, d), dtype=np.float32)
    k = rng.standard_normal((N, d), dtype=np.float32)
    v = rng.standard_normal((N, d), dtype=np.float32)
    do = rng.standard_normal((rows, d), dtype=np.float32)
    scale = d ** -0.5
    r0 = N - rows                     # last rows: a causal sample sees every key
    la = _stock_reference()
    t0 = time.perf_counter()
    if la is not None:
        from burstsim.linalg import Matrix, Vector
        from burstsim.masking import BlockMask
        M = lambda a: Matrix.from_array(a, dtype=np.float32)
        tiles = la.TileSpec(128, 128)
        mask = BlockMask(causal=True) if cfg["causal"] else None
        part = la.local_forward_tiled(M(q), M(k), M(v), scale, tiles, mask, row_offset=r0,
                                      col_offset=0, n_total=N)
        o, lse = part.finalize()
        dst = Vector((do * o.array).sum(1), dtype=np.float32)
        la.local_backward(M(q), M(k), M(v), M(do), lse, dst, scale, tiles, mask, row_offset=r0,
                          col_offset=0, n_total=N)
        kind = "reference"
    else:
        from oracle import burst_oracle as orc
        qpos, kpos = np.arange(r0, N), np.arange(N)
        part = orc.local_forward_tiled(q, k, v, scale, 128, 128, qpos, kpos, cfg["causal"])
        o, lse = part.finalize()
        dst = (do * o).sum(1)
        orc.local_backward(q, k, v, do, lse.astype(np.float32), dst.astype(np.float32), scale,
                           128, 128, qpos, kpos, cfg["causal"])
        kind = "port"
    dt = time.perf_counter() - t0
    # whole step: batch * heads * N query rows (causal: half the pairs on average)
    factor = cfg["batch"] * cfg["heads"] * N / rows * _density(cfg) * (0.5 if cfg["causal"] else 1.0)
    return dt, factor, kind


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        return max(i.get("num_threads", 1) for i in threadpool_info()) or 1
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


def config_dict(cfg, world: int, comm: str):
    """The `config` object of both arms' JSON lines (identical by construction)."""
    B, N, H, D, causal = cfg["batch"], cfg["seq"], cfg["heads"], cfg["d"], cfg["causal"]
    zigzag = causal and world > 1
    n = N // world
    return {"workload": cfg["workload"], "seq": N, "heads": H, "head_dim": D, "batch": B,
            "visible_fraction": _density(cfg) * (0.5 if causal else 1.0),
            "causal": causal, "partition": "zigzag" if zigzag else "contiguous",
            "parallelism": f"ring sp{world}", "comm": comm if world > 1 else None,
            "l2": f"inputs larger than L2 ({B * n * H * D * 2 / 2**30:.2f} GiB per tensor per rank)"}


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_reference_sample(cfg, world, args.ref_rows)
    times = []
    factor, kind = 1.0, "port"
    for _ in range(args.steps):
        dt, factor, kind = cpu_reference_sample(cfg, world, args.ref_rows)
        times.append(dt)
    t_step = statistics.mean(times) * factor
    tokens = cfg["batch"] * cfg["seq"] / t_step
    what = ("stock burstsim.local_attn (baseline/_ref)" if kind == "reference"
            else "oracle port of the reference's tiled kernels")
    sample = (f"{args.ref_rows} query rows x {cfg['seq']} keys x 1 head per step, fwd+bwd, "
              f"{what}, 128x128 tiles, fp32, {statistics.mean(times):.2f} s per sample; "
              f"extrapolated x{factor:.0f} to the whole step")
    line = {"impl": "reference", "metric": METRIC, "value": tokens, "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_step * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(cfg, world, args.comm),
            "extrapolated": True, "sample_rows": args.ref_rows,
            "sample_s_per_step": statistics.mean(times),
            "cpu_baseline": {"value": tokens, "unit": "tokens/s", "cores": cpu_threads(),
                             "kind": kind, "sample": sample},
            "e2e": {"value": tokens, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "tflops_per_gpu": _flops(cfg) / world / t_step / 1e12}
    print(json.dumps(line), flush=True)


def _density(cfg):
    """Fraction of the score matrix a grid mask leaves visible (1 without a mask)."""
    m = cfg.get("mask")
    if not m:
        return 1.0
    return 1.0 - len(m["skip"]) / (m["n_query_blocks"] * m["n_key_blocks"])


def _flops(cfg):
    f = 14.0 * cfg["batch"] * cfg["heads"] * cfg["seq"] ** 2 * cfg["d"] * _density(cfg)
    return f / 2 if cfg["causal"] else f


# ----------------------------------------------------------------- ours

def run_ours(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2403_09347_b200.api import burst_attn_func
    from paper_2403_09347_b200.kernels import CudaKernels
    from paper_2403_09347_b200.schedule import hop_flops

    dev = torch.device("cuda", local_rank)
    B, N, H, D, causal = cfg["batch"], cfg["seq"], cfg["heads"], cfg["d"], cfg["causal"]
    zigzag = causal and world > 1
    if N % (2 * world if zigzag else world):
        raise SystemExit(f"seq {N} not divisible for {world} ranks")
    n = N // world

    class TimedKernels(CudaKernels):
        def __init__(self):
            super().__init__()
            self.on = False
            self.launches = 0
            self.ev = {"fwd": [], "bwd": []}

        def _t(self, kind, flops, fn, stream):
            s = stream if stream is not None else torch.cuda.current_stream()
            if self.on:
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                fn()
                b.record(s)
                self.ev[kind].append((a, b, flops))
            else:
                fn()

        def fwd(self, plan, q, k, v, scale, state, o, lse, first, finalize, stream=None):
            self.launches += 1
            self._t("fwd", hop_flops(plan, B, H, D)[0],
                    lambda: super(TimedKernels, self).fwd(plan, q, k, v, scale, state, o, lse,
                                                          first, finalize, stream), stream)

        def bwd(self, plan, q, k, v, dout, scale, st, dk, dv, accumulate, stream=None):
            self.launches += 1
            self._t("bwd", hop_flops(plan, B, H, D)[1],
                    lambda: super(TimedKernels, self).bwd(plan, q, k, v, dout, scale, st, dk, dv,
                                                          accumulate, stream), stream)

        def fwd_finalize(self, *a, **kw):
            self.launches += 1
            return super().fwd_finalize(*a, **kw)

        def bwd_prepare(self, *a, **kw):
            self.launches += 1
            return super().bwd_prepare(*a, **kw)

        def tl_sum(self, *a, **kw):
            self.launches += 1
            return super().tl_sum(*a, **kw)

        def accumulate(self, *a, **kw):
            self.launches += 2          # one burst_tl_accumulate per dK, dV buffer
            return super().accumulate(*a, **kw)

        def accumulate_dq(self, *a, **kw):
            self.launches += 1
            return super().accumulate_dq(*a, **kw)

        def bwd_finalize(self, st, dk_parts, *a, **kw):
            # burst_bwd_finalize = one tl_rows launch for dQ + one each for dK, dV
            self.launches += 3 if dk_parts else 1
            return super().bwd_finalize(st, dk_parts, *a, **kw)

    kern = TimedKernels()
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    q, k, v, do = (torch.randn(B, n, H, D, device=dev, generator=g, dtype=torch.bfloat16)
                   for _ in range(4))
    for t in (q, k, v):
        t.requires_grad_(True)

    def step(qq, kk, vv, dd, recorders=None):
        o, lse = burst_attn_func(qq, kk, vv, causal=causal, zigzag=zigzag, _kernels=kern,
                                 comm=args.comm, mask=cfg.get("mask"), _recorders=recorders,
                                 deterministic=args.deterministic)
        grads = torch.autograd.grad(o, (qq, kk, vv), dd)
        return o, grads

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step(q, k, v, do)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    kern.on = True
    kern.launches = 0
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        start.record()
        for _ in range(args.steps):
            step(q, k, v, do)
        end.record()
        torch.cuda.synchronize()
        barrier()
    torch.cuda.synchronize()
    kern.on = False
    ms = start.elapsed_time(end) / args.steps
    launches = kern.launches
    # collectives on small host-side values: CUDA tensors for NCCL, CPU for gloo
    cdev = dev if world > 1 and dist.get_backend() == "nccl" else "cpu"
    if world > 1:
        t = torch.tensor([ms], device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()

    def kstats(kind):
        ev = kern.ev[kind]
        if not ev:
            return None, None
        durs = [a.elapsed_time(b) for a, b, _ in ev]
        fl = [f for _, _, f in ev]
        return statistics.mean(durs), statistics.mean(fl)

    bwd_ms, bwd_fl = kstats("bwd")
    fwd_ms, fwd_fl = kstats("fwd")

    # ---- one extra (untimed) traced step: measured hop timeline of every rank's
    # comm and compute streams (trace.py, the reference's ScheduleTrace schema)
    comm_trace = None
    if world > 1:
        from paper_2403_09347_b200.trace import PassRecorder, comm_summary
        recs = (PassRecorder(rank), PassRecorder(rank))
        step(q, k, v, do, recs)
        torch.cuda.synchronize()
        sf, sb = comm_summary(recs[0].events()), comm_summary(recs[1].events())
        vals = torch.tensor([sf["send_us"], sf["hidden_us"], sb["send_us"], sb["hidden_us"],
                             sf["exposed_us"], sb["exposed_us"]],
                            device=cdev, dtype=torch.float64)
        allv = [torch.zeros_like(vals) for _ in range(world)]
        dist.all_gather(allv, vals)
        tot = torch.stack(allv).sum(0).tolist()
        comm_trace = {"fwd_send_us_all_ranks": tot[0], "fwd_hidden_frac": tot[1] / max(tot[0], 1e-9),
                      "bwd_send_us_all_ranks": tot[2], "bwd_hidden_frac": tot[3] / max(tot[2], 1e-9),
                      "fwd_exposed_us_all_ranks": tot[4], "bwd_exposed_us_all_ranks": tot[5],
                      "fwd_stall_hidden_frac": max(0.0, 1 - tot[4] / max(tot[0], 1e-9)),
                      "bwd_stall_hidden_frac": max(0.0, 1 - tot[5] / max(tot[2], 1e-9)),
                      "fwd_bytes_per_rank": recs[0].ledger.bytes_sent_forward,
                      "bwd_bytes_per_rank": recs[1].ledger.bytes_sent_backward,
                      "fwd_GBps_per_rank": recs[0].ledger.bytes_sent_forward
                      / max(tot[0] / world, 1e-9) / 1e3,
                      "bwd_GBps_per_rank": recs[1].ledger.bytes_sent_backward
                      / max(tot[2] / world, 1e-9) / 1e3}
        if args.comm == "ce":
            # host time to post one exchange (device-side flags: no host round trip)
            from paper_2403_09347_b200.api import _transport_for
            hu = sorted(_transport_for(None, "ce").host_us)
            if hu:
                comm_trace["host_us_per_exchange_median"] = hu[len(hu) // 2]
                comm_trace["host_us_per_exchange_max"] = hu[-1]

    # ---- e2e through the public API with pinned host buffers, as a training loop
    # would run it: step i's inputs are copied host->device while step i-1 computes
    # (dO may still be in flight during step i's forward) and step i's results go
    # device->host while step i+1 computes (O already during step i's backward; one
    # stream per copy direction, double-buffered device inputs).  The timed region
    # starts before the first H2D and ends after the last D2H.
    host = [t.detach().cpu().pin_memory() for t in (q, k, v, do)]
    outs = [torch.empty(B, n, H, D, dtype=torch.bfloat16).pin_memory() for _ in range(4)]
    dbuf = [[torch.empty(B, n, H, D, device=dev, dtype=torch.bfloat16) for _ in range(4)]
            for _ in range(2)]
    comp = torch.cuda.current_stream(dev)
    h2d, d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)

    def run_e2e(nsteps, e_start=None, e_stop=None):
        # per buffer: q/k/v landed (the forward may start), dO landed (the backward may)
        ev_qkv = [torch.cuda.Event(), torch.cuda.Event()]
        ev_do = [torch.cuda.Event(), torch.cuda.Event()]
        ev_done = [None, None]
        if e_start is not None:
            e_start.record(h2d)

        def load(i):
            b = dbuf[i % 2]
            if ev_done[i % 2] is not None:
                h2d.wait_event(ev_done[i % 2])     # step i-2 has finished reading b
            with torch.cuda.stream(h2d):
                for dst, src in zip(b[:3], host[:3]):
                    dst.copy_(src, non_blocking=True)
                ev_qkv[i % 2].record(h2d)
                b[3].copy_(host[3], non_blocking=True)
                ev_do[i % 2].record(h2d)

        load(0)
        for i in range(nsteps):
            comp.wait_event(ev_qkv[i % 2])
            qq, kk, vv, dd = dbuf[i % 2]
            qq, kk, vv = (x.detach().requires_grad_(True) for x in (qq, kk, vv))
            o, lse = burst_attn_func(qq, kk, vv, causal=causal, zigzag=zigzag, _kernels=kern,
                                     comm=args.comm, mask=cfg.get("mask"),
                                     deterministic=args.deterministic)
            fwd_done = torch.cuda.Event()
            fwd_done.record(comp)
            d2h.wait_event(fwd_done)               # O leaves while the backward runs
            with torch.cuda.stream(d2h):
                o.record_stream(d2h)
                outs[0].copy_(o.detach(), non_blocking=True)
            comp.wait_event(ev_do[i % 2])
            gq, gk, gv = torch.autograd.grad(o, (qq, kk, vv), dd)
            done = torch.cuda.Event()
            done.record(comp)
            ev_done[i % 2] = done
            if i + 1 < nsteps:
                load(i + 1)
            d2h.wait_event(done)
            with torch.cuda.stream(d2h):
                for dst, src in zip(outs[1:], (gq, gk, gv)):
                    src.record_stream(d2h)
                    dst.copy_(src.detach(), non_blocking=True)
        if e_stop is not None:
            d2h.wait_stream(h2d)
            e_stop.record(d2h)

    # the same K steps as the device-timed region: the fill (step 0's q/k/v H2D) and the
    # drain (the last step's dQ/dK/dV D2H) are paid once per K steps, as in a training loop
    e2e_steps = max(2, args.steps)
    run_e2e(2)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    run_e2e(e2e_steps, e0, e1)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_ms], device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = t.item()
    tensor_bytes = B * n * H * D * 2

    if rank != 0:
        return
    peaks = _peaks()
    peak_burst = peaks.get("bf16_tflops", 1590.0)
    peak_sus = peaks.get("bf16_tflops_sustained", 1400.0)
    peak_src = "MEASURED_PEAKS.json" if peaks else "fallback (B200_PROFILING.md)"
    tokens = B * N / (ms / 1e3)
    tflops_gpu = _flops(cfg) / world / (ms / 1e3) / 1e12
    traffic = traffic_fwd = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = tr.get(f"{args.config}_g{world}", {}).get("lao_bwd")
        traffic_fwd = tr.get(f"{args.config}_g{world}", {}).get("lao_fwd")
    except Exception:  # noqa: BLE001
        pass
    roof = None
    if bwd_ms:
        ach = bwd_fl / (bwd_ms / 1e3) / 1e12
        roof = {"bound": "tensor", "kernel": "lao_bwd4_kernel<128> (LAO backward, sm_100a tcgen05, key-tile pairs in 2-CTA clusters sharing Q/dO by TMA multicast, 2 P/dS warpgroups, TMA bulk dQ reduction)",
                "achieved": ach, "peak": peak_sus, "unit": "TFLOP/s", "frac": ach / peak_sus,
                "peak_kind": f"bf16 sustained ({peak_src}); kernel runs inside a long step",
                "frac_of_burst_peak": ach / peak_burst, "traffic": traffic,
                "flops_per_launch": bwd_fl, "ms_per_launch": bwd_ms}
        if fwd_ms:
            fa = fwd_fl / (fwd_ms / 1e3) / 1e12
            roof["lao_fwd"] = {"achieved": fa, "frac": fa / peak_sus,
                               "frac_of_burst_peak": fa / peak_burst, "ms_per_launch": fwd_ms,
                               "flops_per_launch": fwd_fl, "traffic": traffic_fwd}
    cpu = None
    if world == 1 and not args.skip_cpu:
        dt, factor, kind = cpu_reference_sample(cfg, 1, args.cpu_rows)
        ct = dt * factor
        cpu = {"value": B * N / ct, "unit": "tokens/s", "cores": cpu_threads(), "kind": kind,
               "sample": f"{args.cpu_rows} query rows x {N} keys x 1 head fwd+bwd ("
                         + ("stock burstsim.local_attn" if kind == "reference" else
                            "oracle port of the reference tiled algorithm")
                         + f", numpy fp32) in {dt:.2f}s, extrapolated x{factor:.0f}",
               "extrapolated": True, "tflops": _flops(cfg) / ct / 1e12}
    comm = None
    if world > 1:
        from paper_2403_09347_b200.ring import ring_comm_bytes
        fb, bb = ring_comm_bytes(n, B, H, D, world, 2, causal, zigzag)
        comm = {"bytes_sent_per_rank_per_step": fb + bb,
                "avg_GBps_over_step": (fb + bb) / (ms / 1e3) / 1e9,
                "measured": comm_trace}
    line = {
        "metric": METRIC, "value": tokens, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded N(0,1) q/k/v/dO)",
        "config": dict(config_dict(cfg, world, args.comm),
                       **({"deterministic": True} if args.deterministic else {})),
        "tflops_per_gpu": tflops_gpu, "tc_peak_frac": tflops_gpu / peak_sus,
        "tc_peak_frac_of_burst": tflops_gpu / peak_burst,
        "e2e": {"value": B * N / (e2e_ms / 1e3), "unit": "tokens/s",
                "h2d_bytes_per_step": 4 * tensor_bytes, "d2h_bytes_per_step": 4 * tensor_bytes,
                "ms_per_step": e2e_ms, "steps": e2e_steps,
                "api": "burst_attn_func + autograd; pinned host buffers, H2D of step i+1 and "
                       "D2H of step i on two copy streams overlapping compute (dO lands during "
                       "the forward, O leaves during the backward); the window spans the same "
                       "K steps as the device timing and includes the pipeline fill (step 0's "
                       "q/k/v) and drain (the last dQ/dK/dV)"},
        "roofline": roof, "cpu_baseline": cpu, "clocks": clk.summary(),
        "gpu_launches": launches, "comm": comm,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-rows", type=int, default=1024,
                    help="query rows of the reference arm's per-step CPU sample (~3 s each)")
    ap.add_argument("--cpu-rows", type=int, default=3072,
                    help="query rows of the cpu_baseline sample in our line (~10 s of CPU work)")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "ce"],
                    help="ring transport at N>1: NCCL send/recv, or copy engines over CUDA IPC")
    ap.add_argument("--deterministic", action="store_true",
                    help="bit-reproducible backward (ordered dQ reductions)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    import torch
    # Test hook: BURST_BENCH_ONE_GPU=1 puts every rank on device 0 (exercises the N > 1
    # code paths on a one-GPU box; use with BURST_BENCH_BACKEND=gloo and --comm ce,
    # since NCCL refuses two ranks on one device).  Not a measurement configuration.
    if os.environ.get("BURST_BENCH_ONE_GPU") == "1":
        local_rank = 0
    torch.cuda.set_device(local_rank)
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = os.environ.get("BURST_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    if args.gpus != world and world > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    run_ours(args, cfg, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
