"""Measured-trace export and causality linting (simulator schemas,
reference sim.py:459-599). CPU tests drive the linter with synthetic traces,
including the tamper cases the reference tests its own linter with
(pkg/tests/test_sim.py:194-219); the GPU test traces a real step."""
import json

import pytest
import torch

from paper_2411_01075_b200 import GpuAssignment, ModelSpec, TrainPlan, assign_unit_shards
from paper_2411_01075_b200.data import rank_tokens
from paper_2411_01075_b200.model import ARCHS
from paper_2411_01075_b200.trace import (StepTracer, TraceEvent, lint_measured_trace,
                                         per_layer_metrics, trace_to_chrome, trace_to_jsonl)


def _good_trace(blocks=3, l=2):
    ev, t = [], 0.0
    for u in range(1, blocks + 1):
        ev.append(TraceEvent("g0", "allgather", u, 0, "fwd", t, t + 0.5))
        t += 0.5
        for j in range(1, l + 1):
            ev.append(TraceEvent("g0", "fwd_compute", u, j, "fwd", t, t + 1.0))
            t += 1.0
    for u in range(blocks, 0, -1):
        for j in range(1, l + 1):
            ev.append(TraceEvent("g0", "recompute", u, j, "bwd", t, t + 1.0))
            ev.append(TraceEvent("g0", "bwd_compute", u, j, "bwd", t + 1.0, t + 3.0))
            t += 3.0
        ev.append(TraceEvent("g0", "reducescatter", u, 0, "bwd", t, t + 0.5))
    return ev


def test_clean_trace_lints_clean_and_exports(tmp_path):
    ev = _good_trace()
    assert lint_measured_trace(ev, 3) == []
    fwd, bwd = per_layer_metrics(ev, 3)
    assert fwd == pytest.approx(2.5) and bwd == pytest.approx(6.0)
    trace_to_jsonl(ev, tmp_path / "t.jsonl")
    rows = [json.loads(x) for x in (tmp_path / "t.jsonl").read_text().splitlines()]
    assert set(rows[0]) == {"gpu", "kind", "unit", "microbatch", "phase", "start_ms", "end_ms"}
    trace_to_chrome(ev, tmp_path / "t.json")
    doc = json.loads((tmp_path / "t.json").read_text())
    assert any(e.get("ph") == "X" for e in doc["traceEvents"])


@pytest.mark.parametrize("tamper", ["early_forward", "overlap", "early_rs", "bwd_before_ra"])
def test_tampered_traces_are_flagged(tamper):
    ev = _good_trace()
    if tamper == "early_forward":       # forward before its all-gather finished
        ev = [TraceEvent(e.gpu_id, e.kind, e.unit, e.microbatch, e.phase,
                         e.start_ms - 0.4 if e.kind == "fwd_compute" and e.unit == 2 and
                         e.microbatch == 1 else e.start_ms, e.end_ms) for e in ev]
    elif tamper == "overlap":
        ev.append(TraceEvent("g0", "fwd_compute", 1, 3, "fwd", 1.0, 1.8))
    elif tamper == "early_rs":
        ev = [TraceEvent(e.gpu_id, e.kind, e.unit, e.microbatch, e.phase,
                         e.start_ms - 2.0 if e.kind == "reducescatter" else e.start_ms,
                         e.end_ms) for e in ev]
    elif tamper == "bwd_before_ra":
        ev = [TraceEvent(e.gpu_id, e.kind, e.unit, e.microbatch, e.phase,
                         e.start_ms - 0.6 if e.kind == "bwd_compute" else e.start_ms,
                         e.end_ms) for e in ev]
    assert lint_measured_trace(ev, 3), tamper


def _at(ev, kind, unit, mb):
    return next(e for e in ev if (e.kind, e.unit, e.microbatch) == (kind, unit, mb))


@pytest.mark.parametrize("case", ["clean", "late_fwd_prefetch", "late_grad_prefetch",
                                  "early_grad_offload"])
def test_offload_rules(case):
    """The simulator's offload residency rules (sim.py:226-338) on the measured
    trace: forward-phase input prefetches, activation-gradient offload and
    prefetch."""
    ev = _good_trace()
    f = _at(ev, "fwd_compute", 2, 1)
    b2 = _at(ev, "bwd_compute", 2, 1)
    b3 = _at(ev, "bwd_compute", 3, 1)
    shift = {"late_fwd_prefetch": 0.3, "late_grad_prefetch": 0.3,
             "early_grad_offload": -0.3}.get(case, 0.0)
    ev.append(TraceEvent("g0", "prefetch_act", 2, 1, "fwd", f.start_ms - 0.5,
                         f.start_ms + (shift if case == "late_fwd_prefetch" else 0.0)))
    ev.append(TraceEvent("g0", "prefetch_grad", 2, 1, "bwd", b2.start_ms - 0.5,
                         b2.start_ms + (shift if case == "late_grad_prefetch" else 0.0)))
    t0 = b3.end_ms + (shift if case == "early_grad_offload" else 0.0)
    ev.append(TraceEvent("g0", "offload_grad", 3, 1, "bwd", t0, t0 + 0.2))
    problems = lint_measured_trace(ev, 3)
    assert (problems == []) == (case == "clean"), problems


@pytest.mark.gpu
def test_real_step_trace_is_causal(cuda, tmp_path):
    from paper_2411_01075_b200.step import UnevenFSDPTrainer
    arch = ARCHS["tiny_gpt"]
    model = ModelSpec(arch.layers, arch.unit_params, 4)
    plan = TrainPlan((GpuAssignment("g0", 2, 2, 4, 1.0, 0.0, float(model.state_bytes)),),
                     1.0, 1.0, 2.0 * arch.layers, False, assign_unit_shards([1.0], model))
    tr = UnevenFSDPTrainer(arch, plan, 0, device=cuda)
    tr.init_params(0)
    tok = torch.from_numpy(rank_tokens(plan, 0, arch.seq, arch.vocab, 1, 0)).to(cuda)
    tr.step(tok)
    tr.tracer = StepTracer("g0")
    tr.step(tok)
    ev = tr.tracer.collect()
    kinds = {e.kind for e in ev}
    assert {"fwd_compute", "recompute", "bwd_compute", "head", "optimizer"} <= kinds
    assert sum(e.kind == "fwd_compute" and e.unit > 0 for e in ev) == arch.layers * 2
    assert lint_measured_trace(ev, arch.layers) == []
    fwd, bwd = per_layer_metrics(ev, arch.layers)
    assert fwd > 0 and bwd > 0
    trace_to_jsonl(ev, tmp_path / "step.jsonl")


def test_boundary_residency_ledger_rules():
    """trace.boundary_residency follows the reference ledger (sim.py:226-322):
    a unit-major schedule of L units x l microbatches holds l + 1 boundary
    items without offload; with the simulator's offload hand-off (prefetch
    lands as the previous offload drains) it holds 2."""
    from paper_2411_01075_b200.trace import TraceEvent, boundary_residency
    L, l = 3, 4
    ev, t = [], 0.0
    for u in range(1, L + 1):
        for j in range(1, l + 1):
            ev.append(TraceEvent("g", "fwd_compute", u, j, "fwd", t, t + 1.0))
            t += 1.0
    for u in range(L, 0, -1):
        for j in range(1, l + 1):
            ev.append(TraceEvent("g", "recompute", u, j, "bwd", t, t + 1.0))
            ev.append(TraceEvent("g", "bwd_compute", u, j, "bwd", t + 1.0, t + 3.0))
            t += 3.0
    assert boundary_residency(ev, L)["g"] == l + 1
    # offload: every forward/backward item prefetched during the previous compute,
    # outputs drained during the next one (transfer time = compute time / 2)
    off = [e for e in ev]
    for e in ev:
        if e.kind == "fwd_compute":
            off.append(TraceEvent("g", "offload_act", e.unit, e.microbatch, "fwd", e.end_ms,
                                  e.end_ms + 0.5))
            if e.unit > 1:
                off.append(TraceEvent("g", "prefetch_act", e.unit, e.microbatch, "fwd",
                                      e.start_ms - 0.5, e.start_ms))
        if e.kind == "bwd_compute" and e.unit > 1:
            off.append(TraceEvent("g", "prefetch_act", e.unit, e.microbatch, "bwd",
                                  e.start_ms - 1.5, e.start_ms - 1.0))
    assert boundary_residency(off, L)["g"] == 2
