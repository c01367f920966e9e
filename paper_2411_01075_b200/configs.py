"""The benchmark configurations of BASELINE.json, as reference-schema
documents (cluster JSON core.py:298-327, profile JSON core.py:362-376, model
JSON core.py:344-355) for emulated heterogeneous B200 clusters.

B200s are homogeneous, so a "tier" is an emulated GPU class: a fraction of
the SMs (CUDA green context, `emulate.py`) and an HBM budget (memory-fraction
cap). Profiles here are ANALYTIC first-order models of a B200 tier (FLOPs at
an assumed sustained bf16 rate scaled by the SM fraction, plus a per-
microbatch launch floor); `profiler.py` replaces them with measured tables
in the same schema. The planner consumes either unchanged.
"""
from __future__ import annotations

import dataclasses
import json
from dataclasses import dataclass
from pathlib import Path

from .core import ClusterSpec, ModelSpec, TrainPlan, cluster_from_dict, model_from_dict, profile_from_dict
from .model import ARCHS, ArchSpec
from .perf import ClusterPerf, FitError, fit_perf_model
from .planner import dp_optimize
from .sharding import assign_unit_shards

GIB = 1 << 30
SUSTAINED_TFLOPS = 500.0      # assumed achieved bf16 rate of the model GEMMs on a full B200
LAUNCH_FLOOR_MS = 0.08        # per microbatch per unit (kernel launches, small GEMM tails)
NVLINK_GBS = 700.0            # assumed per-GPU collective bandwidth for the comm profile

# tier name -> (SM fraction, HBM budget GiB)
TIERS: dict[str, tuple[float, float]] = {
    "b200": (1.0, 160.0),
    "b200_3q": (0.75, 96.0),
    "b200_half": (0.5, 64.0),
    "b200_quarter": (0.25, 32.0),
    # tight budgets for the Llama config (forces single-owner/mixed shards)
    "b200_tight": (1.0, 40.0),
    "b200_small": (0.5, 20.0),
}


def _unit_flops_fwd(arch: ArchSpec, m: int) -> float:
    tok = m * arch.seq
    return 2.0 * arch.unit_params * tok + 4.0 * arch.seq * arch.d * tok


def _act_bytes_per_sample(arch: ArchSpec) -> float:
    s, d = arch.seq, arch.d
    checkpoints = (arch.layers + 1) * s * d * 2
    transient = 24 * s * d * 2 + (s * arch.heads * s * 2 if arch.kind == "bert" else 0)
    logits = s * arch.vocab * (2 + 4 + 4)
    return checkpoints + transient + logits


def tier_profile(arch: ArchSpec, tier: str, max_m: int = 8) -> dict:
    frac, _ = TIERS[tier]
    rate = SUSTAINED_TFLOPS * 1e12 * frac / 1e3          # FLOP per ms
    fwd = [[m, LAUNCH_FLOOR_MS + _unit_flops_fwd(arch, m) / rate] for m in range(1, max_m + 1)]
    bwd = [[m, 2 * LAUNCH_FLOOR_MS + 2 * _unit_flops_fwd(arch, m) / rate]
           for m in range(1, max_m + 1)]
    base = (2 * arch.unit_params * (2 + 4) + arch.root_params * (2 + 4)) / GIB + 1.5
    per = _act_bytes_per_sample(arch) / GIB
    mem = [[m, base + per * m] for m in range(1, max_m + 1)]
    return {"profile_key": tier, "fwd_ms": fwd, "bwd_ms": bwd, "compute_mem_gib": mem}


def cluster_doc(arch: ArchSpec, tiers: list[str], mem_cap_fraction: float = 0.8,
                memory_gib: dict[str, float] | None = None) -> dict:
    """Cluster JSON (core.py:298-327); `memory_gib` overrides a tier's HBM budget."""
    ag = arch.unit_params * 2 / (NVLINK_GBS * 1e6)
    rs = arch.unit_params * 4 / (NVLINK_GBS * 1e6)
    mem = {t: TIERS[t][1] for t in tiers} | dict(memory_gib or {})
    return {"gpus": [{"id": f"{t}-{i}", "memory_gib": mem[t], "profile_key": t}
                     for i, t in enumerate(tiers)],
            "comm": {"allgather_ms": ag, "reducescatter_ms": rs, "uneven_overhead": 0.15},
            "mem_cap_fraction": mem_cap_fraction}


@dataclass(frozen=True)
class BenchConfig:
    name: str
    arch: str
    tiers: tuple[str, ...]        # 8-GPU tier list; N GPUs take the first N
    batch_per_gpu: int            # global batch = batch_per_gpu * N (weak scaling)
    description: str
    # per-config HBM budgets (GiB) overriding configs.TIERS for the named tiers
    memory_gib: tuple[tuple[str, float], ...] = ()


CONFIGS: dict[str, BenchConfig] = {
    "tiny_gpt": BenchConfig("tiny_gpt", "tiny_gpt", ("b200", "b200_half") * 4, 6,
                            "tiny GPT (4 layers, d=256), 2:1 emulated ranks"),
    "gpt2_small": BenchConfig("gpt2_small", "gpt2_small", ("b200", "b200_half") * 4, 64,
                              "GPT-2 small uneven-FSDP, emulated 2:1 compute and memory"),
    # the three smaller tiers get HBM budgets below their compute memory at the
    # batch they can process, so the planner gives them l_i > 1 (layered GA,
    # PAPER.md:377-386) and puts the whole training state on the full tier
    "bert_large": BenchConfig("bert_large", "bert_large",
                              ("b200", "b200_3q", "b200_half", "b200_quarter") * 2, 48,
                              "BERT-large bf16, 4-tier emulated cluster, layered GA",
                              (("b200_3q", 2.5), ("b200_half", 2.0), ("b200_quarter", 1.5))),
    "llama_1b3": BenchConfig("llama_1b3", "llama_1b3",
                             ("b200_tight", "b200_small") * 4, 16,
                             "Llama-style 1.3B, tight per-rank HBM caps"),
}


@dataclass(frozen=True)
class Job:
    config: BenchConfig
    arch: ArchSpec
    cluster: ClusterSpec
    model: ModelSpec
    perf: ClusterPerf
    plan: TrainPlan
    profile_docs: tuple[dict, ...]


def perf_from_docs(docs) -> ClusterPerf:
    models = {}
    for d in docs:
        c, m = profile_from_dict(d)
        models[c.profile_key] = fit_perf_model(c, m)
    return ClusterPerf(models)


MEASURED_DIR = Path(__file__).resolve().parent / "profiles_b200"


def measured_profiles(name: str) -> dict[str, dict] | None:
    """Profiles measured on a B200 by tools/profile_tiers.py, if committed."""
    p = MEASURED_DIR / f"{name}.json"
    if not p.exists():
        return None
    return {d["profile_key"]: d for d in json.loads(p.read_text())["profiles"]}


def planner_model(arch: ArchSpec, global_batch: int) -> dict:
    """Model JSON (core.py:344-355) the planner sees: the root unit's
    parameters (embeddings, final norm, tied head: 31% of GPT-2 small) are
    amortised into params_per_layer, as the reference fixtures do
    (fixtures/model_bert_large.json), so state_bytes = 16 (L U + E)
    (core.py:151-154) covers the whole training state the ranks hold."""
    ppl = -(-(arch.layers * arch.unit_params + arch.root_params) // arch.layers)
    return {"layers": arch.layers, "params_per_layer": ppl, "global_batch": global_batch}


def build_job(name: str, n_gpus: int, global_batch: int | None = None,
              measured: bool = False) -> Job:
    """Cluster, model, fitted perf models and the planner's plan for a config.
    measured=True uses the B200-measured tier profiles when available (the
    analytic ones otherwise)."""
    cfg = CONFIGS[name]
    arch = ARCHS[cfg.arch]
    tiers = list(cfg.tiers[:n_gpus]) if n_gpus <= len(cfg.tiers) else \
        [cfg.tiers[i % len(cfg.tiers)] for i in range(n_gpus)]
    meas = measured_profiles(name) if measured else None
    docs = tuple(meas[t] if meas and t in meas else tier_profile(arch, t)
                 for t in sorted(set(tiers)))
    if meas:
        try:
            perf_from_docs(docs)
        except FitError:   # launch-bound tables with no linear tail: keep the analytic model
            docs = tuple(tier_profile(arch, t) for t in sorted(set(tiers)))
    cluster = cluster_from_dict(cluster_doc(arch, tiers, memory_gib=dict(cfg.memory_gib)))
    batch = global_batch if global_batch is not None else cfg.batch_per_gpu * n_gpus
    model = model_from_dict(planner_model(arch, batch))
    perf = perf_from_docs(docs)
    plan = dp_optimize(cluster, model, perf)
    # the flat layout shards the real units (U params each; the root unit gets the
    # same ratios in layout.root_shard_plan), not the amortised planning unit
    plan = dataclasses.replace(plan, unit_shards=assign_unit_shards(
        [a.state_ratio for a in plan.assignments], arch.model_spec(batch)))
    return Job(cfg, arch, cluster, model, perf, plan, docs)
