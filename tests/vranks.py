"""Virtual-rank harness: N ranks of the fused symmetric collectives on ONE GPU.

The fused kernels (csrc/hetstep_symm.cu) address every rank's copy of the
symmetric buffer through ``het_symm_t.peer_base[j]``; they never ask where
that memory lives. Here one allocation holds N equal copies (rank j's copy at
``base + j * stride``) and N descriptors differ only in ``rank``. All N ranks
run as ONE cooperative launch (``het_symm_virtual``: CTA b of rank r at
blockIdx r * ctas + b, the same kernel bodies and in-kernel barriers as N real
launches), so every CTA is co-resident by construction -- kernels that wait on
one another are never separate launches on one GPU (B200_PROFILING.md). The
driver's 1-GPU test run thereby exercises the NR = 2 / 4 / 8 specialisations,
the peer, relay and helper routes and both reduce-scatters against the oracle.

This is test infrastructure (it measures nothing: a "link" is local HBM).
"""
from __future__ import annotations

import ctypes
from typing import Sequence

import torch

from paper_2411_01075_b200 import hetstep as K

ALIGN = 256


class VirtualGroup:
    def __init__(self, n: int, regions: Sequence[tuple[str, int, torch.dtype]],
                 device: torch.device, ctas: int | None = None):
        if not 1 <= n <= K.HET_MAX_RANKS:
            raise ValueError("1..8 virtual ranks")
        lib = K.load()
        self.n, self.device = n, device
        self.offsets, pos = {}, 0
        self.regions = list(regions)
        for name, numel, dtype in regions:
            self.offsets[name] = pos
            esz = torch.tensor([], dtype=dtype).element_size()
            pos += (numel * esz + ALIGN - 1) // ALIGN * ALIGN
        self.signal_off = pos
        per_rank = pos + int(lib.het_symm_signal_bytes())
        self.stride = (per_rank + 4095) // 4096 * 4096
        self.raw = torch.zeros(n * self.stride, dtype=torch.uint8, device=device)
        base = self.raw.data_ptr()
        self.desc = []
        for r in range(n):
            d = K.HetSymm()
            d.nranks, d.rank = n, r
            for j in range(n):
                d.peer_base[j] = base + j * self.stride
            d.mc_base = 0                       # one GPU: no NVLS multicast object
            d.signal_off = self.signal_off
            self.desc.append(d)
        # one cooperative grid of n * ctas CTAs (het_symm_virtual refuses more than fit)
        sms = torch.cuda.get_device_properties(device).multi_processor_count
        self.ctas = ctas if ctas is not None else max(1, min(32, sms // n))
        self.epoch = [0, 0]
        self.dev_base: list[int] | None = None
        torch.cuda.synchronize(device)

    def set_device_base(self, base: Sequence[int]) -> None:
        """Seed every rank's device epoch base (het_symm_epoch_set) and switch the
        launches to device epochs; the host counters continue from `base`."""
        lib = K.load()
        for r in range(self.n):
            for ch in range(K.SYMM_CHANNELS):
                K._check(lib.het_symm_epoch_set(ctypes.byref(self.desc[r]), ch, int(base[ch]),
                                                torch.cuda.current_stream(self.device).cuda_stream),
                         "het_symm_epoch_set")
        self.epoch = list(base)
        self.dev_base = list(base)

    def add_device_base(self, ch: int, delta: int) -> None:
        """het_symm_epoch_add on every rank: launches numbered from the new base."""
        lib = K.load()
        for r in range(self.n):
            K._check(lib.het_symm_epoch_add(ctypes.byref(self.desc[r]), ch, int(delta),
                                            torch.cuda.current_stream(self.device).cuda_stream),
                     "het_symm_epoch_add")
        self.dev_base[ch] += delta

    def signal_words(self, r: int, count: int) -> torch.Tensor:
        """The first `count` uint32 barrier slots of rank r (channel 0, start
        barrier, CTA 0: one per source rank)."""
        return K.region_tensor(self.raw, r * self.stride + self.signal_off, count, torch.int32)

    def view(self, r: int, name: str) -> torch.Tensor:
        """Rank r's copy of a region (its own version counter, like the real
        workspace's regions: hetstep.region_tensor)."""
        for nm, numel, dtype in self.regions:
            if nm == name:
                return K.region_tensor(self.raw, r * self.stride + self.offsets[name], numel,
                                       dtype)
        raise KeyError(name)

    def _run(self, op: int, region: str, byte_off: int, srcs, outs, counts, offsets,
             weights=None, channel: int = 0, end_barrier: bool = True,
             policy: int = K.SYMM_AUTO, stage_off: int = 0) -> None:
        lib, n = K.load(), self.n
        self.epoch[channel] += 1
        # device-epoch mode (set_device_base): the launch passes its offset from the
        # per-rank device base, flagged EPOCH_DEVICE, as a captured step does
        ep = self.epoch[channel] if self.dev_base is None else \
            K.EPOCH_DEVICE | (self.epoch[channel] - self.dev_base[channel])
        descs = (K.HetSymm * n)(*self.desc)
        src_p = (ctypes.c_void_p * n)(*[(t.data_ptr() if t is not None and t.numel() else None)
                                        for t in srcs])
        out_p = (ctypes.c_void_p * n)(*[(t.data_ptr() if t is not None and t.numel() else None)
                                        for t in outs])
        w = (ctypes.c_float * n)(*[float(x) for x in weights]) if weights is not None else None
        torch.cuda.synchronize(self.device)
        K._check(lib.het_symm_virtual(op, n, descs, src_p, out_p, K._i64(counts), K._i64(offsets),
                                      byte_off, w, ep, channel,
                                      int(end_barrier), int(policy), int(stage_off), self.ctas,
                                      torch.cuda.current_stream(self.device).cuda_stream),
                 "het_symm_virtual")

    def allgather_pack(self, srcs: Sequence[torch.Tensor], region: str, elem_off: int,
                       counts: Sequence[int], offsets: Sequence[int], policy: int = K.SYMM_AUTO
                       ) -> None:
        self._run(K.OP_AG, region, self.offsets[region] + 2 * elem_off, srcs, [None] * self.n,
                  counts, offsets, channel=0, policy=policy)

    def reduce_scatter(self, region: str, elem_off: int, outs: Sequence[torch.Tensor],
                       counts: Sequence[int], offsets: Sequence[int], end_barrier: bool = True,
                       policy: int = K.SYMM_AUTO) -> None:
        self._run(K.OP_RS, region, self.offsets[region] + 4 * elem_off, [None] * self.n, outs,
                  counts, offsets, channel=1, end_barrier=end_barrier, policy=policy)

    def reduce_scatter_bf16(self, region: str, elem_off: int, outs: Sequence[torch.Tensor],
                            counts: Sequence[int], offsets: Sequence[int],
                            weights: Sequence[float], end_barrier: bool = True,
                            policy: int = K.SYMM_AUTO, stage: str | None = None) -> None:
        stage_off = self.offsets[stage] + 4 * elem_off if stage is not None else 0
        self._run(K.OP_RS_BF16, region, self.offsets[region] + 2 * elem_off, [None] * self.n,
                  outs, counts, offsets, weights=weights, channel=1, end_barrier=end_barrier,
                  policy=policy, stage_off=stage_off)
