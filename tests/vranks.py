"""Virtual-rank harness: N ranks of the fused symmetric collectives on ONE GPU.

The fused kernels (csrc/hetstep_symm.cu) address every rank's copy of the
symmetric buffer through ``het_symm_t.peer_base[j]``; they never ask where
that memory lives. Here one allocation holds N equal copies (rank j's copy at
``base + j * stride``), N descriptors differ only in ``rank``, and rank r's
kernel is launched on its own stream. The N launches run concurrently, meet
at the same in-kernel CTA-pairwise barriers as on N GPUs (peer stores and
loads are plain HBM accesses here), and produce the same bytes, so the
driver's 1-GPU test run exercises the NR = 2 / 4 / 8 specialisations, the
peer and relay all-gathers and both reduce-scatters against the oracle.

Co-residency: every barrier needs CTA b of all N launches resident at once.
``ctas * N`` is kept below one CTA per SM (148), so they always are, and the
barriers cannot time out unless a rank is deliberately left out.

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
        # one CTA per SM at most across all virtual ranks (co-residency of every barrier)
        sms = torch.cuda.get_device_properties(device).multi_processor_count
        self.ctas = ctas if ctas is not None else max(1, min(32, (sms - 4) // n))
        if self.ctas * n > sms:
            raise ValueError("ctas * n exceeds one CTA per SM: barriers could deadlock")
        self.streams = [torch.cuda.Stream(device=device) for _ in range(n)]
        self.epoch = [0, 0]
        torch.cuda.synchronize(device)

    def view(self, r: int, name: str) -> torch.Tensor:
        """Rank r's copy of a region (its own version counter, like the real
        workspace's regions: hetstep.region_tensor)."""
        for nm, numel, dtype in self.regions:
            if nm == name:
                return K.region_tensor(self.raw, r * self.stride + self.offsets[name], numel,
                                       dtype)
        raise KeyError(name)

    def _launch(self, fn, ranks) -> None:
        torch.cuda.synchronize(self.device)     # inputs written on the default stream
        for r in ranks:
            fn(r, self.streams[r].cuda_stream)
        torch.cuda.synchronize(self.device)

    def allgather_pack(self, srcs: Sequence[torch.Tensor], region: str, elem_off: int,
                       counts: Sequence[int], offsets: Sequence[int], policy: int = K.SYMM_AUTO,
                       ranks: Sequence[int] | None = None) -> None:
        self.epoch[0] += 1
        lib, c, o = K.load(), K._i64(counts), K._i64(offsets)
        byte_off = self.offsets[region] + 2 * elem_off

        def go(r, st):
            src = srcs[r].data_ptr() if srcs[r].numel() else None
            K._check(lib.het_symm_allgather_pack(ctypes.byref(self.desc[r]), src, byte_off, c, o,
                                                 self.epoch[0], 0, policy, self.ctas, st),
                     "het_symm_allgather_pack")
        self._launch(go, range(self.n) if ranks is None else ranks)

    def reduce_scatter(self, region: str, elem_off: int, outs: Sequence[torch.Tensor],
                       counts: Sequence[int], offsets: Sequence[int], end_barrier: bool = True,
                       policy: int = K.SYMM_AUTO) -> None:
        self.epoch[1] += 1
        lib, c, o = K.load(), K._i64(counts), K._i64(offsets)
        byte_off = self.offsets[region] + 4 * elem_off

        def go(r, st):
            out = outs[r].data_ptr() if outs[r].numel() else None
            K._check(lib.het_symm_reduce_scatter(ctypes.byref(self.desc[r]), byte_off, out, c, o,
                                                 self.epoch[1], 1, int(end_barrier), policy,
                                                 self.ctas, st),
                     "het_symm_reduce_scatter")
        self._launch(go, range(self.n))

    def reduce_scatter_bf16(self, region: str, elem_off: int, outs: Sequence[torch.Tensor],
                            counts: Sequence[int], offsets: Sequence[int],
                            weights: Sequence[float], end_barrier: bool = True,
                            policy: int = K.SYMM_AUTO, stage: str | None = None) -> None:
        self.epoch[1] += 1
        lib, c, o = K.load(), K._i64(counts), K._i64(offsets)
        byte_off = self.offsets[region] + 2 * elem_off
        stage_off = self.offsets[stage] + 4 * elem_off if stage is not None else 0
        w = (ctypes.c_float * len(weights))(*[float(x) for x in weights])

        def go(r, st):
            out = outs[r].data_ptr() if outs[r].numel() else None
            K._check(lib.het_symm_reduce_scatter_bf16(ctypes.byref(self.desc[r]), byte_off, out,
                                                      c, o, w, self.epoch[1], 1,
                                                      int(end_barrier), policy, stage_off,
                                                      self.ctas, st),
                     "het_symm_reduce_scatter_bf16")
        self._launch(go, range(self.n))


# ---------------------------------------------------------------------------
# virtual ranks of the whole train step: N trainers in N threads on one GPU

class VirtualRankGroup:
    """Host-side agreement of N trainers running in N threads of one process
    (the step's DistGroup stand-in): sum_ranks is a barrier + shared sum."""

    def __init__(self, n: int, timeout: float = 300.0):
        import threading
        self.n = n
        # a rank that dies breaks the barrier for the others instead of hanging them
        self._bar = threading.Barrier(n, timeout=timeout)
        self._lock = threading.Lock()
        self._vals: list[int] = []
        self._out = 0

    def sum_ranks(self, value: int) -> int:
        with self._lock:
            self._vals.append(int(value))
        if self._bar.wait() == 0:
            with self._lock:
                self._out = sum(self._vals)
                self._vals = []
        self._bar.wait()
        return self._out

    def barrier(self) -> None:
        self._bar.wait()


class _Handle:
    def __init__(self, group: VirtualRankGroup, device):
        self.group, self.device = group, device

    def barrier(self) -> None:
        torch.cuda.current_stream(self.device).synchronize()
        self.group.barrier()


class VirtualSymmWorkspace(K.SymmWorkspace):
    """Rank r's view of a VirtualGroup allocation, with SymmWorkspace's methods:
    the trainer issues the same fused kernels as on N GPUs (peer route; no NVLS
    multicast object on one GPU)."""

    def __init__(self, vg: VirtualGroup, rank: int, group: VirtualRankGroup,
                 policy: int = K.SYMM_AUTO):
        self.offsets = dict(vg.offsets)
        self.signal_off = vg.signal_off
        self.multicast = False
        self.desc = vg.desc[rank]
        self.views = {name: vg.view(rank, name) for name, _, _ in vg.regions}
        self.epoch = [0, 0]
        self.ctas = vg.ctas
        self.policy = policy
        self.handle = _Handle(group, vg.device)


def run_ranks(n: int, fn, group: VirtualRankGroup | None = None) -> list:
    """fn(r) for r in 0..n-1 in n threads; re-raises the first exception (a
    failing rank aborts the group's barrier so the others fail too)."""
    import threading
    out, err = [None] * n, [None] * n

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:          # noqa: BLE001 (reported below)
            err[r] = e
            if group is not None:
                group._bar.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out
