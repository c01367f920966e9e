"""Measured per-rank traces of the real train step in the reference
simulator's schemas, plus a causality linter for them.

The reference simulates one iteration and exports it as JSONL (one event per
line: gpu, kind, unit, microbatch, phase, start_ms, end_ms — sim.py:549-561)
or as a Chrome/Perfetto trace (pid = GPU, tid = stream, sim.py:564-599), and
`lint_trace` (sim.py:459-542) checks the schedule's causality. Here the same
event kinds are timed on the GPU with CUDA events on the stream that runs
them (compute, all-gather, reduce-scatter), relative to a step-start event,
so a real step can be inspected with the same tools and linted with the same
rules:
  * stream exclusivity: compute events of one GPU never overlap;
  * fwd_compute(u, j) starts after the all-gather that delivered unit u;
  * recompute(u, j) starts after unit u is resident for the backward (its
    backward all-gather, or the forward one for the two units this step keeps
    resident — DESIGN.md §3);
  * bwd_compute(u, j) starts after recompute(u, j);
  * with activation offload: the H2D and D2H copy streams are each exclusive;
    offload_act(u, j) starts after fwd_compute(u, j) (the forward that consumed
    or produced the checkpoint); fwd_compute(u, j) / recompute(u, j) start
    after their forward- / backward-phase prefetch_act(u, j) landed;
    offload_grad(u, j) starts after the bwd_compute(u, j) that produced it
    (the head's, for unit 0); bwd_compute(u, j) starts after prefetch_grad(u, j)
    landed (sim.py:226-338);
  * reducescatter(u) starts after the rank's last bwd_compute(u, .).
Units are 1-indexed like the simulator; the root unit (embeddings/head) is
unit 0. Cross-rank rules of the simulator (identical collective windows on
every GPU) do not apply to measured per-rank clocks and are not checked.
"""
from __future__ import annotations

import json
from contextlib import contextmanager
from dataclasses import dataclass
from pathlib import Path
from typing import Iterable

import torch

COMPUTE_KINDS = ("fwd_compute", "recompute", "bwd_compute", "head", "embed_bwd", "optimizer")
COLLECTIVE_KINDS = ("allgather", "reducescatter")
H2D_KINDS = ("prefetch_act", "prefetch_grad")
D2H_KINDS = ("offload_act", "offload_grad")
_TID = {"compute": 0, "h2d": 1, "d2h": 2, "network": 3}
EPS = 1e-3          # ms; event timestamps have ~0.5 us resolution


@dataclass(frozen=True)
class TraceEvent:
    gpu_id: str
    kind: str
    unit: int
    microbatch: int
    phase: str
    start_ms: float
    end_ms: float

    @property
    def duration_ms(self) -> float:
        return self.end_ms - self.start_ms


class StepTracer:
    """Collects CUDA-event spans during one UnevenFSDPTrainer.step()."""

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self._spans: list[tuple[str, int, int, str, torch.cuda.Event, torch.cuda.Event]] = []
        self._t0: torch.cuda.Event | None = None

    def begin(self, stream) -> None:
        self._spans.clear()
        self._t0 = torch.cuda.Event(enable_timing=True)
        self._t0.record(stream)

    @contextmanager
    def span(self, kind: str, unit: int, microbatch: int, phase: str, stream):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        try:
            yield
        finally:
            b.record(stream)
            self._spans.append((kind, unit, microbatch, phase, a, b))

    def collect(self) -> list[TraceEvent]:
        torch.cuda.synchronize()
        out = [TraceEvent(self.gpu_id, k, u, j, ph, self._t0.elapsed_time(a),
                          self._t0.elapsed_time(b)) for k, u, j, ph, a, b in self._spans]
        return sorted(out, key=lambda e: (e.start_ms, e.kind, e.phase, e.unit, e.microbatch))


def trace_to_jsonl(events: Iterable[TraceEvent], path: str | Path) -> None:
    with open(path, "w") as fh:
        for e in events:
            fh.write(json.dumps({"gpu": e.gpu_id, "kind": e.kind, "unit": e.unit,
                                 "microbatch": e.microbatch, "phase": e.phase,
                                 "start_ms": e.start_ms, "end_ms": e.end_ms},
                                sort_keys=True) + "\n")


def _stream_of(kind: str) -> str:
    if kind in H2D_KINDS:
        return "h2d"
    if kind in D2H_KINDS:
        return "d2h"
    return "network" if kind in COLLECTIVE_KINDS else "compute"


def trace_to_chrome(events: Iterable[TraceEvent], path: str | Path) -> None:
    events = list(events)
    gpus = sorted({e.gpu_id for e in events})
    pid = {g: i for i, g in enumerate(gpus)}
    out = []
    for g, p in pid.items():
        out.append({"name": "process_name", "ph": "M", "pid": p, "tid": 0, "args": {"name": g}})
        for s, t in _TID.items():
            out.append({"name": "thread_name", "ph": "M", "pid": p, "tid": t, "args": {"name": s}})
    for e in events:
        tid = _TID[_stream_of(e.kind)] + (1 if e.kind == "reducescatter" else 0) * 10
        out.append({"name": f"{e.kind} u{e.unit}" + (f" j{e.microbatch}" if e.microbatch else ""),
                    "cat": e.phase, "ph": "X", "ts": e.start_ms * 1000.0,
                    "dur": e.duration_ms * 1000.0, "pid": pid[e.gpu_id], "tid": tid,
                    "args": {"unit": e.unit, "microbatch": e.microbatch}})
    Path(path).write_text(json.dumps({"traceEvents": out, "displayTimeUnit": "ms"},
                                     sort_keys=True) + "\n")


def lint_measured_trace(events: Iterable[TraceEvent], blocks: int) -> list[str]:
    """Per-GPU causality checks of a measured step (rules in the module doc)."""
    problems: list[str] = []
    by_gpu: dict[str, list[TraceEvent]] = {}
    for e in events:
        if e.end_ms < e.start_ms - EPS or e.start_ms < -EPS:
            problems.append(f"bad interval on {e.gpu_id} {e.kind} u{e.unit} j{e.microbatch}")
        by_gpu.setdefault(e.gpu_id, []).append(e)
    for g, evs in by_gpu.items():
        for kinds, label in ((COMPUTE_KINDS, "compute"), (H2D_KINDS, "h2d"), (D2H_KINDS, "d2h")):
            ss = sorted((e for e in evs if e.kind in kinds), key=lambda e: e.start_ms)
            for a, b in zip(ss, ss[1:]):
                if b.start_ms < a.end_ms - EPS:
                    problems.append(f"{label} overlap on {g}: {a.kind} u{a.unit} / "
                                    f"{b.kind} u{b.unit}")
        ag = {(e.phase, e.unit): e for e in evs if e.kind == "allgather"}
        idx = {(e.kind, e.unit, e.microbatch): e for e in evs if e.kind in COMPUTE_KINDS}
        pf = {(e.kind, e.unit, e.microbatch, e.phase): e for e in evs if e.kind in H2D_KINDS}

        def landed(kind, e, phase, label):
            c = pf.get((kind, e.unit, e.microbatch, phase))
            if c and e.start_ms < c.end_ms - EPS:
                problems.append(f"{label} u{e.unit} j{e.microbatch} on {g} starts before its "
                                f"{kind}")
        last_bwd: dict[int, float] = {}
        for e in evs:
            if e.kind == "fwd_compute":
                c = ag.get(("fwd", e.unit))
                if c and e.start_ms < c.end_ms - EPS:
                    problems.append(f"F u{e.unit} j{e.microbatch} on {g} starts before its allgather")
                landed("prefetch_act", e, "fwd", "F")
            elif e.kind == "recompute":
                c = ag.get(("bwd", e.unit)) or ag.get(("fwd", e.unit))
                if c and e.start_ms < c.end_ms - EPS:
                    problems.append(f"RA u{e.unit} j{e.microbatch} on {g} starts before its allgather")
                landed("prefetch_act", e, "bwd", "RA")
            elif e.kind == "offload_act":
                f = idx.get(("fwd_compute", e.unit, e.microbatch))
                if f and e.start_ms < f.end_ms - EPS:
                    problems.append(f"offload_act u{e.unit} j{e.microbatch} on {g} starts "
                                    "before its forward finished")
            elif e.kind == "offload_grad":
                b = idx.get(("head" if e.unit == 0 else "bwd_compute", e.unit, e.microbatch))
                if b and e.start_ms < b.end_ms - EPS:
                    problems.append(f"offload_grad u{e.unit} j{e.microbatch} on {g} starts "
                                    "before the backward that produced it")
            elif e.kind == "bwd_compute":
                ra = idx.get(("recompute", e.unit, e.microbatch))
                if ra and e.start_ms < ra.end_ms - EPS:
                    problems.append(f"B u{e.unit} j{e.microbatch} on {g} starts before its recompute")
                landed("prefetch_grad", e, "bwd", "B")
                last_bwd[e.unit] = max(last_bwd.get(e.unit, 0.0), e.end_ms)
        for e in evs:
            if e.kind == "reducescatter" and e.unit in last_bwd and \
                    e.start_ms < last_bwd[e.unit] - EPS:
                problems.append(f"reducescatter u{e.unit} on {g} starts before its last backward")
        for u in range(1, blocks + 1):
            if ("fwd_compute", u, 1) not in idx and any(e.kind == "fwd_compute" for e in evs):
                problems.append(f"unit {u} never ran forward on {g}")
    return problems


def per_layer_metrics(events: Iterable[TraceEvent], blocks: int) -> tuple[float, float]:
    """Measured per-layer forward / backward period (the simulator's
    definition, sim.py:412-425): max gap between consecutive units' first
    microbatch starts, per GPU, maximised over GPUs."""
    events = list(events)
    fwd = bwd = 0.0
    for g in {e.gpu_id for e in events}:
        fs = {e.unit: e.start_ms for e in events
              if e.gpu_id == g and e.kind == "fwd_compute" and e.microbatch == 1}
        bs = {e.unit: e.start_ms for e in events
              if e.gpu_id == g and e.kind == "recompute" and e.microbatch == 1}
        for u in range(1, blocks):
            if u in fs and u + 1 in fs:
                fwd = max(fwd, fs[u + 1] - fs[u])
            if u in bs and u + 1 in bs:
                bwd = max(bwd, bs[u] - bs[u + 1])
    return fwd, bwd


def _peak(intervals) -> float:
    """Max simultaneous size over [start, end) intervals; frees sort before
    allocations at the same timestamp (the reference's _peak, sim.py:102-119)."""
    pts = []
    for a, b, size in intervals:
        if b > a:
            pts.append((a, size))
            pts.append((b, -size))
    pts.sort(key=lambda p: (p[0], p[1]))
    level = peak = 0.0
    for _, d in pts:
        level += d
        peak = max(peak, level)
    return peak


def boundary_residency(events: Iterable[TraceEvent], blocks: int) -> dict[str, float]:
    """Peak resident boundary activations per GPU, in items (one microbatch's
    unit-boundary tensor), from a MEASURED trace with the reference's ledger
    rules (sim.py:226-322; peak_activation_memory sim.py:440-442):

      without offload  the output of unit u-1 for microbatch j lives from its
                       forward until unit u's forward of j consumed it; in the
                       backward the checkpointed input of u > 1 lives through
                       recompute(u, j) .. bwd_compute(u, j); the last unit's
                       outputs drain at its first backward;
      with offload     a prefetched input lives from its H2D landing until its
                       consumer (forward or backward) ends; a produced output
                       lives until its D2H landed.

    The reference asserts (l + 1) items without offload and 2 with it
    (test_acceptance.py:157-186)."""
    out: dict[str, float] = {}
    events = list(events)
    for g in sorted({e.gpu_id for e in events}):
        ev = {(e.kind, e.phase, e.unit, e.microbatch): e for e in events if e.gpu_id == g}
        offload = any(k[0] == "offload_act" for k in ev)
        js = sorted({k[3] for k in ev if k[0] == "fwd_compute"})
        iv = []
        for u in range(1, blocks + 1):
            for j in js:
                f = ev.get(("fwd_compute", "fwd", u, j))
                b = ev.get(("bwd_compute", "bwd", u, j))
                if f is None or b is None:
                    continue
                if offload:
                    pf = ev.get(("prefetch_act", "fwd", u, j))
                    if u > 1 and pf is not None:
                        iv.append((pf.end_ms, f.end_ms, 1.0))
                    oa = ev.get(("offload_act", "fwd", u, j))
                    if oa is not None:
                        iv.append((f.end_ms, oa.end_ms, 1.0))
                    pb = ev.get(("prefetch_act", "bwd", u, j))
                    if u > 1 and pb is not None:
                        iv.append((pb.end_ms, b.end_ms, 1.0))
                else:
                    if u > 1:
                        prev = ev.get(("fwd_compute", "fwd", u - 1, j))
                        if prev is not None:
                            iv.append((prev.end_ms, f.end_ms, 1.0))
                        rc = ev.get(("recompute", "bwd", u, j))
                        start = rc.start_ms if rc is not None else b.start_ms
                        iv.append((start, b.end_ms, 1.0))
                    if u == blocks:
                        iv.append((f.end_ms, b.start_ms, 1.0))
        out[g] = _peak(iv)
    return out
