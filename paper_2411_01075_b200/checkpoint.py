"""Sharded checkpoint / resume of the uneven training state, keyed by the
plan's UnitShardPlan (the reference persists only plan
JSON, core.py:482-492).

Layout on disk (one directory per checkpoint):
  plan.json            the TrainPlan (reference schema, core.py:405-432)
  meta.json            step count, unit sizes, per-rank range tables
  rank{i}.pt           rank i's fp32 master / exp_avg / exp_avg_sq ranges, one
                       tensor per unit (only the rank's [offsets, +counts) slice)

Each rank writes only what it owns: a save is embarrassingly parallel and
moves 12 B per owned parameter. Loading under the same shard tables reads
the rank's own file; loading under a DIFFERENT plan (other ratios, other
rank count) re-shards: every requested range is assembled from the saved
ranks whose ranges overlap it, so a job can resume on a re-planned cluster.
"""
from __future__ import annotations

import json
import os
from pathlib import Path

import torch

from .core import InputError, TrainPlan, load_plan, save_plan
from .layout import RankLayout

STATE = ("p32", "m32", "v32")


def _tables(layout: RankLayout) -> dict:
    return {"counts": [list(c) for c in layout.counts],
            "offsets": [list(o) for o in layout.offsets],
            "unit_params": layout.unit_params, "root_params": layout.root_params,
            "nranks": layout.nranks}


def save_shards(path: str | Path, layout: RankLayout, buffers: dict[str, torch.Tensor],
                step: int, plan: TrainPlan | None = None, barrier=None) -> None:
    """Write this rank's ranges of every state buffer (flat local layout).
    Every file is written to a temporary name and renamed into place; with
    `barrier` (a cross-rank barrier callable) rank 0 writes meta.json only
    after every rank's file is in place, so meta.json marks a complete save."""
    d = Path(path)
    d.mkdir(parents=True, exist_ok=True)
    per_unit = {}
    for name in STATE:
        buf = buffers[name]
        per_unit[name] = [buf[off:off + cnt].detach().to("cpu", torch.float32).clone()
                          for off, cnt in (layout.local_range(u)
                                           for u in range(layout.blocks + 1))]
    _atomic(d / f"rank{layout.rank}.pt",
            lambda tmp: torch.save({"rank": layout.rank, "step": step, "state": per_unit}, tmp))
    if barrier is not None:
        barrier()            # every rank file is complete before meta.json names them
    if layout.rank == 0:
        if plan is not None:
            _atomic(d / "plan.json", lambda tmp: save_plan(plan, tmp))
        # meta.json last: a reader that sees it sees a complete checkpoint
        _atomic(d / "meta.json", lambda tmp: Path(tmp).write_text(
            json.dumps({"step": step, **_tables(layout)}, indent=1)))


def _atomic(dst: Path, write) -> None:
    """write(tmp) then rename over dst (POSIX rename is atomic on one filesystem)."""
    tmp = dst.with_name(f".{dst.name}.tmp{os.getpid()}")
    write(tmp)
    os.replace(tmp, dst)


def load_shards(path: str | Path, layout: RankLayout) -> tuple[dict[str, list[torch.Tensor]], int]:
    """This rank's ranges (per unit, per state buffer) under `layout`,
    re-sharding from the saved tables when they differ."""
    d = Path(path)
    meta = json.loads((d / "meta.json").read_text())
    if meta["unit_params"] != layout.unit_params or meta["root_params"] != layout.root_params \
            or len(meta["counts"]) != layout.blocks + 1:
        raise InputError("checkpoint was written for a different model shape")
    missing = [r for r in range(meta["nranks"]) if not (d / f"rank{r}.pt").exists()]
    if missing:
        raise InputError(f"checkpoint is incomplete: missing rank files {missing}")
    same = meta["counts"] == [list(c) for c in layout.counts]
    cache: dict[int, dict] = {}

    def saved(r: int) -> dict:
        if r not in cache:
            f = d / f"rank{r}.pt"
            if not f.exists():
                raise InputError(f"checkpoint is missing {f.name}")
            cache[r] = torch.load(f, map_location="cpu", weights_only=True)
        return cache[r]

    out: dict[str, list[torch.Tensor]] = {name: [] for name in STATE}
    if same:
        st = saved(layout.rank)["state"]
        for name in STATE:
            out[name] = list(st[name])
        return out, int(meta["step"])
    for u in range(layout.blocks + 1):
        lo = layout.offsets[u][layout.rank]
        hi = lo + layout.counts[u][layout.rank]
        parts = {name: torch.empty(hi - lo, dtype=torch.float32) for name in STATE}
        for r in range(meta["nranks"]):
            s_lo = meta["offsets"][u][r]
            s_hi = s_lo + meta["counts"][u][r]
            a, b = max(lo, s_lo), min(hi, s_hi)
            if a >= b:
                continue
            st = saved(r)["state"]
            for name in STATE:
                parts[name][a - lo:b - lo] = st[name][u][a - s_lo:b - s_lo]
        for name in STATE:
            out[name].append(parts[name])
    return out, int(meta["step"])


def save_trainer(trainer, path: str | Path) -> None:
    """Checkpoint an UnevenFSDPTrainer (every rank calls this)."""
    if trainer.cuda:
        torch.cuda.synchronize(trainer.device)
    barrier = None
    if trainer.N > 1:
        import torch.distributed as dist
        if dist.is_initialized():
            barrier = dist.barrier
    save_shards(path, trainer.L, {n: getattr(trainer, n) for n in STATE}, trainer.steps,
                trainer.plan, barrier=barrier)


def load_trainer(trainer, path: str | Path) -> int:
    """Resume an UnevenFSDPTrainer from a checkpoint written under any plan of
    the same model; refreshes the bf16 shadow. Returns the step count."""
    parts, step = load_shards(path, trainer.L)
    for name in STATE:
        buf = getattr(trainer, name)
        for u, t in enumerate(parts[name]):
            off, cnt = trainer.L.local_range(u)
            buf[off:off + cnt].copy_(t.to(buf.device))
    trainer.steps = step
    trainer.refresh_shadow()
    return step


def checkpoint_plan(path: str | Path) -> TrainPlan:
    return load_plan(Path(path) / "plan.json")
