"""Heterogeneity emulation on homogeneous B200s (north_star: "per-rank HBM
budgets are set with a memory-fraction cap, and per-rank SM partitions are
set with CUDA green contexts").

A rank's tier comes from the cluster spec: its `memory_gib` (the emulated
physical HBM, not the planner's 0.8 effective capacity) becomes a cap on
the torch caching allocator (`set_per_process_memory_fraction`), and the
tier's SM fraction (configs.TIERS) becomes a CUDA green context holding that
many SMs; the rank's compute stream is created inside it, so every model and
owned kernel launched on it is confined to the partition. Collective streams
stay outside the partition: NVLink bandwidth is not partitioned on real
mixed clusters either, which matches the reference's cluster-wide
communication scalars (core.py:70-82).

Caveats (documented, not hidden): NCCL's internal buffers, cuBLAS workspaces
and the symmetric-memory workspace are allocated outside the caching
allocator and so outside the cap.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from .configs import TIERS
from .core import ClusterSpec, InputError

SM_GRANULE = 8     # green-context SM partitions are taken in groups of SMs


@dataclass
class TierEmulation:
    tier: str
    sm_fraction: float
    num_sms: int
    memory_cap_bytes: int
    stream: torch.cuda.Stream | None   # compute stream (inside the green context)
    green: object | None

    def describe(self) -> dict:
        return {"tier": self.tier, "sm_fraction": self.sm_fraction, "num_sms": self.num_sms,
                "memory_cap_gib": self.memory_cap_bytes / 2 ** 30,
                "green_context": self.green is not None}


def emulate_tier(cluster: ClusterSpec, rank: int, device: torch.device, *,
                 sm_partition: bool = True, memory_cap: bool = True) -> TierEmulation:
    gpu = cluster.gpus[rank]
    if gpu.profile_key not in TIERS:
        raise InputError(f"unknown tier {gpu.profile_key!r} for emulation")
    frac, _ = TIERS[gpu.profile_key]
    props = torch.cuda.get_device_properties(device)
    total_sms = props.multi_processor_count
    # the emulated GPU's physical HBM: the planner's mem_cap_fraction headroom
    # (core.py:143-144) stays available at run time for what its memory model
    # omits (allocator fragmentation, the N>1 gather/accumulate buffers)
    cap = int(gpu.memory_capacity)
    if memory_cap:
        torch.cuda.set_per_process_memory_fraction(min(1.0, cap / props.total_memory), device)
    green, stream, nsm = None, None, total_sms
    if sm_partition and frac < 1.0:
        nsm = max(SM_GRANULE, int(round(frac * total_sms / SM_GRANULE)) * SM_GRANULE)
        green = torch.cuda.GreenContext.create(nsm, device.index)
        raw = green.Stream()
        stream = raw if isinstance(raw, torch.cuda.Stream) else torch.cuda.Stream(
            stream_id=raw.stream_id, device_index=raw.device_index, device_type=raw.device_type)
        # persistent grids of the owned kernels sized for the partition (one wave
        # fills nsm SMs instead of 148 x k CTAs queueing in it)
        from . import hetstep as K
        K.set_sm_budget(nsm)
    return TierEmulation(gpu.profile_key, frac, nsm, cap, stream, green)
