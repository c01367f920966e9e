"""B200 profiler: measured per-tier profiles in the reference's schema
(profile_from_dict, core.py:362-376), feeding the planner (
PAPER.md:632-634 "profiles a few training iterations for each batch size
from 1 to B, fitting linear models").

For an emulated tier (SM fraction via a green context, configs.TIERS) and
microbatch sizes m = 1..max_m it measures, on one GPU:
  fwd_ms[m]  one transformer unit's forward on [m, seq, d] bf16 activations
  bwd_ms[m]  step-calibrated backward: the measured whole 1-GPU step at
             microbatch m over L, minus the unit's forward and its
             recompute (calibrate_bwd), so head / embedding / AdamW time is
             in the planner's per-layer model; calibrate=False keeps the
             unit's backward alone (the planner adds the recompute as
             recompute_multiplier * fwd, planner.py:132)
  compute_mem_gib[m]  peak allocator bytes of a full 1-GPU train step with
             microbatch m minus the sharded training state (16 B/param +
             the 2 B bf16 shadow) — the paper's M_compute = M - M_state
             (PAPER.md:543), affine in m (perf.py:136-144).
Latencies are medians of CUDA-event-timed repetitions on the tier's stream.
"""
from __future__ import annotations

import statistics

import torch

from .configs import TIERS
from .core import GpuAssignment, ModelSpec, TrainPlan
from .model import ArchSpec, block_forward, init_flat, views
from .sharding import assign_unit_shards

GIB = 1 << 30


def _tier_stream(tier: str, device: torch.device):
    frac, _ = TIERS[tier]
    if frac >= 1.0:
        return torch.cuda.Stream(device=device), None
    total = torch.cuda.get_device_properties(device).multi_processor_count
    nsm = max(8, int(round(frac * total / 8)) * 8)
    green = torch.cuda.GreenContext.create(nsm, device.index)
    raw = green.Stream()
    s = raw if isinstance(raw, torch.cuda.Stream) else torch.cuda.Stream(
        stream_id=raw.stream_id, device_index=raw.device_index, device_type=raw.device_type)
    return s, green


def _time(fn, stream, reps: int) -> float:
    with torch.cuda.stream(stream):
        for _ in range(2):
            fn()
        out = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            out.append(a.elapsed_time(b))
    return statistics.median(out)


def unit_latencies(arch: ArchSpec, tier: str, ms: list[int], device: torch.device,
                   reps: int = 9) -> tuple[list[float], list[float]]:
    stream, green = _tier_stream(tier, device)
    gen = torch.Generator(device=device).manual_seed(0)
    flat = init_flat(arch.unit_layout(), gen, device).to(torch.bfloat16)
    params = {k: v.requires_grad_(True) for k, v in views(flat, arch.unit_layout()).items()}
    plist = list(params.values())
    fwd, bwd = [], []
    for m in ms:
        with torch.cuda.stream(stream):
            x = torch.randn(m, arch.seq, arch.d, device=device, dtype=torch.bfloat16)
            dy = torch.randn_like(x)

        def f():
            with torch.no_grad():
                block_forward(arch, params, x)

        holder = {}

        def prep():
            xi = x.detach().requires_grad_(True)
            holder["y"] = block_forward(arch, params, xi)
            holder["x"] = xi

        def b():
            torch.autograd.grad(holder["y"], plist + [holder["x"]], dy)

        fwd.append(_time(f, stream, reps))
        # backward alone: forward outside the timed region, then the graph's backward
        with torch.cuda.stream(stream):
            times = []
            for _ in range(reps + 2):
                prep()
                a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                b()
                e.record(stream)
                e.synchronize()
                times.append(a.elapsed_time(e))
        bwd.append(statistics.median(times[2:]))
    torch.cuda.synchronize(device)
    del green
    return fwd, bwd


def step_latencies(arch: ArchSpec, tier: str, ms: list[int], device: torch.device,
                   reps: int = 3) -> list[float]:
    """Device time of one whole 1-GPU train step (eager, as multi-rank steps
    run: embedding, every unit's forward / recompute / backward, the head,
    accumulate, AdamW) at microbatch m, l = 1, on the tier's SM partition."""
    from .data import rank_tokens
    from .step import UnevenFSDPTrainer
    stream, green = _tier_stream(tier, device)
    out = []
    with torch.cuda.stream(stream):
        for m in ms:
            model = ModelSpec(arch.layers, arch.unit_params, m)
            plan = TrainPlan((GpuAssignment("prof", m, 1, m, 1.0, 0.0,
                                            float(model.state_bytes)),),
                             1.0, 1.0, 2.0 * arch.layers, False, assign_unit_shards([1.0], model))
            tr = UnevenFSDPTrainer(arch, plan, 0, device=device)
            tr.init_params(0)
            tok = torch.from_numpy(rank_tokens(plan, 0, arch.seq, arch.vocab, 0, 0)).to(device)
            out.append(_time(lambda: tr.step(tok), stream, reps))
            del tr, tok
    torch.cuda.synchronize(device)
    del green
    return out


def calibrate_bwd(arch: ArchSpec, fwd: list[float], step: list[float],
                  recompute_multiplier: float = 1.0) -> list[float]:
    """Per-layer backward entries that make the planner's latency model
    (planner.per_gpu_layer_latency, Eqs. 2-3: L * (l F + l (B + rec F)))
    reproduce the measured whole step at l = 1:
        B'(m) = step(m) / L - (1 + rec) F(m).
    The head, the embedding backward, the accumulate and AdamW, which the
    reference's per-layer model has no term for, are thereby amortised over
    the L units exactly as the reference fixtures amortise the embedding
    parameters into params_per_layer (fixtures/model_bert_large.json)."""
    L = arch.layers
    out = []
    for f, st in zip(fwd, step):
        out.append(max(st / L - (1.0 + recompute_multiplier) * f, 1e-3))
    return out


def compute_memory(arch: ArchSpec, ms: list[int], device: torch.device) -> list[float]:
    """Peak allocator bytes of one real 1-GPU step per microbatch size, minus
    the sharded state; GiB."""
    from .data import rank_tokens
    from .step import UnevenFSDPTrainer
    out = []
    for m in ms:
        model = ModelSpec(arch.layers, arch.unit_params, m)
        plan = TrainPlan((GpuAssignment("prof", m, 1, m, 1.0, 0.0, float(model.state_bytes)),),
                         1.0, 1.0, 2.0 * arch.layers, False, assign_unit_shards([1.0], model))
        torch.cuda.synchronize(device)
        torch.cuda.empty_cache()
        base = torch.cuda.memory_allocated(device)
        tr = UnevenFSDPTrainer(arch, plan, 0, device=device)
        tr.init_params(0)
        state = torch.cuda.memory_allocated(device) - base
        tok = torch.from_numpy(rank_tokens(plan, 0, arch.seq, arch.vocab, 0, 0)).to(device)
        tr.step(tok)
        torch.cuda.synchronize(device)
        torch.cuda.reset_peak_memory_stats(device)
        tr.step(tok)
        torch.cuda.synchronize(device)
        peak = torch.cuda.max_memory_allocated(device) - base
        out.append(max(peak - state, 1) / GIB)
        del tr, tok
    return out


def profile_tier(arch: ArchSpec, tier: str, device: torch.device, max_m: int = 8,
                 mem: list[float] | None = None, calibrate: bool = True) -> dict:
    """Profile entry of one tier. calibrate=True (the bench's profiles): the
    backward entries are step-calibrated (calibrate_bwd) so the planner's
    predicted iteration matches the measured whole step."""
    ms = list(range(1, max_m + 1))
    fwd, bwd = unit_latencies(arch, tier, ms, device)
    if calibrate:
        bwd = calibrate_bwd(arch, fwd, step_latencies(arch, tier, ms, device))
    if mem is None:
        mem = compute_memory(arch, ms, device)
    # the schema requires strictly increasing memory in m (core.py:200-203)
    for i in range(1, len(mem)):
        mem[i] = max(mem[i], mem[i - 1] * (1 + 1e-9) + 1e-9)
    return {"profile_key": tier,
            "fwd_ms": [[m, float(v)] for m, v in zip(ms, fwd)],
            "bwd_ms": [[m, float(v)] for m, v in zip(ms, bwd)],
            "compute_mem_gib": [[m, float(v)] for m, v in zip(ms, mem)]}
