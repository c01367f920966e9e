"""The train-step entry point: one Cephalo layered-gradient-accumulation
iteration on one rank (one process per GPU).

Schedule (the reference's executable spec, sim.py:342-368):

  FWD  AG(root), AG(unit 0)                                  [ag stream]
       for u in 0..L-1:  prefetch AG(u+1) into the other buffer once unit
                         u-1 has released it                  [ag stream]
                         all l_i microbatches through unit u, keeping only
                         the unit-boundary activations (checkpoints; with
                         offload_activations they go to pinned host memory)
       head: loss_k and dL/dh_L of microbatch k right behind the last unit's
       forward; root grads accumulate
  BWD  for u in L-1..0:  prefetch AG(u-1) (units L-1 and L-2 are still
                         resident from the forward: no re-gather)
                         for each microbatch: recompute unit u (skipped for
                         the last unit when l_i == 1: its forward graph is
                         kept), backward, het_accumulate(acc_u, grads,
                         w = m_i/B)  (kernel 4; l_i <= 1 plans group units:
                         pairs under collectives, the whole backward on one
                         GPU) then RS(acc_u -> rank's fp32 grad shard)  [rs stream]
                         unit 0's backward feeds het_embedding_grad straight
                         into the root accumulator; RS(root)
  OPT  one het_adamw over the rank's whole flat shard (kernel 5), writing the
       bf16 shadow only when some unit's all-gather goes through NCCL

Collectives are routed per unit (hetstep.route_collective): the fused
symmetric-memory kernels (pack + all-gather from the fp32 master; switch or
peer reduction straight into the fp32 shard) or NCCL rings.

Eq. 1 weighting (gradcheck.py:30-46) is the w = m_i/B pre-scale inside
het_accumulate, so RS is a plain SUM; when every rank has l_i <= 1, fused-route
units instead cross the wire as unscaled bf16 gradients and the reduce-scatter
applies every rank's weight and the cast (het_symm_reduce_scatter_bf16). Idle
ranks (m_i = 0, core.py:224-226) skip compute but still take part in every
AG/RS with zero contributions. On one GPU the unit views point straight into
the bf16 shadow and the accumulator is the grad shard itself: no collectives,
no copies.
"""
from __future__ import annotations

import contextlib
from dataclasses import dataclass, field

import torch

from . import hetstep as K
from .core import InputError, TrainPlan
from .layout import RankLayout
from .model import (ArchSpec, block_forward, embed_forward, head_value_and_grad, init_flat,
                    segment_offsets, views)


@dataclass(frozen=True)
class AdamWConfig:
    lr: float = 1e-3
    betas: tuple[float, float] = (0.9, 0.95)
    eps: float = 1e-8
    weight_decay: float = 0.1


@dataclass
class StepTimers:
    """CUDA events around the owned kernels (enabled for roofline runs)."""
    enabled: bool = False
    external: bool = False     # events recorded inside a CUDA-graph capture
    adamw: list = field(default_factory=list)
    accumulate: list = field(default_factory=list)
    gather: list = field(default_factory=list)

    def pair(self, kind: str, nbytes: float):
        """Start/end events for one launch moving `nbytes` algorithmic bytes."""
        if not self.enabled:
            return None, None
        a = torch.cuda.Event(enable_timing=True, external=self.external)
        b = torch.cuda.Event(enable_timing=True, external=self.external)
        getattr(self, kind).append((a, b, nbytes))
        return a, b

    def reset(self) -> None:
        self.adamw.clear()
        self.accumulate.clear()
        self.gather.clear()

    def summary(self, kind: str) -> dict:
        """launches, total ms, algorithmic bytes and GB/s over the recorded launches."""
        ev = getattr(self, kind)
        ms = [a.elapsed_time(b) for a, b, _ in ev]
        nbytes = sum(x for _, _, x in ev)
        tot = sum(ms)
        return {"launches": len(ev), "ms_total": tot, "ms_mean": tot / len(ev) if ev else 0.0,
                "bytes_total": nbytes,
                "bytes_per_launch": nbytes / len(ev) if ev else 0.0,
                "gbs": nbytes / (tot * 1e-3) / 1e9 if tot > 0 else None}


class _NoStream:
    """Stand-in for CUDA streams/events when a test drives the schedule on CPU
    with injected kernels; the real kernels reject CPU tensors, so this is not
    a compute fallback."""
    cuda_stream = 0

    def wait_event(self, ev) -> None:
        pass

    def wait_stream(self, other) -> None:
        pass

    def record(self, stream=None) -> None:
        pass


class DistGroup:
    """Host-side agreement between the ranks of one step (torch.distributed
    default group: plumbing). A test may pass any object with the same
    `sum_ranks` to drive several ranks from one process (tests/vranks.py)."""

    def __init__(self, dev: torch.device):
        self.dev = dev

    def sum_ranks(self, value: int) -> int:
        """Sum of an integer over the default process group (CPU tensor under gloo)."""
        import torch.distributed as dist
        on_cpu = dist.get_backend() == "gloo"
        t = torch.tensor([int(value)], dtype=torch.int32, device="cpu" if on_cpu else self.dev)
        dist.all_reduce(t)
        return int(t.item())


class UnevenFSDPTrainer:
    """Per-rank state (uneven flat shards in HBM) plus the step driver."""

    def __init__(self, arch: ArchSpec, plan: TrainPlan, rank: int, *,
                 comm_ag: K.Comm | None = None, comm_rs: K.Comm | None = None,
                 opt: AdamWConfig = AdamWConfig(), device: torch.device | None = None,
                 algo: int = K.ALGO_AUTO, group_name: str | None = None, symm_ctas: int = 32,
                 offload_activations: bool = False, offload_schedule: str = "reference",
                 check_routes: bool = True,
                 bf16_wire: bool = True, group=None, symm_workspace=None):
        """group: host-side rank agreement (default DistGroup over torch.distributed);
        symm_workspace: a pre-built symmetric workspace with this trainer's regions
        (default: allocated through torch symmetric memory when algo = ALGO_SYMM)."""
        if plan.unit_shards is None or plan.unit_shards.units != arch.layers:
            raise InputError("plan unit_shards must have one row per transformer block")
        self.arch, self.plan, self.rank, self.opt, self.algo = arch, plan, rank, opt, algo
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.cuda = self.device.type == "cuda"
        if self.cuda:
            K.load()
        self.L = RankLayout.from_plan(plan, arch.unit_params, arch.root_params, rank)
        self.N = self.L.nranks
        if self.N > 1 and (comm_ag is None or comm_rs is None) and symm_workspace is None:
            raise InputError("multi-rank plan needs the AG and RS communicators")
        self._group = group if group is not None else (DistGroup(self.device)
                                                      if self.N > 1 else None)
        self.comm_ag, self.comm_rs = comm_ag, comm_rs
        a = plan.assignments[rank]
        self.m, self.l = a.microbatch, a.num_microbatches
        self.B = plan.total_batch
        self.w = self.m / self.B
        dev, n = self.device, self.L.local_len
        self.p32 = torch.zeros(n, dtype=torch.float32, device=dev)
        self.g32 = torch.zeros(n, dtype=torch.float32, device=dev)
        self.m32 = torch.zeros(n, dtype=torch.float32, device=dev)
        self.v32 = torch.zeros(n, dtype=torch.float32, device=dev)
        self.p16 = torch.zeros(n, dtype=torch.bfloat16, device=dev)
        U, E = arch.unit_params, arch.root_params
        self.symm = None
        self.symm_error = None
        if self.N > 1 and symm_workspace is not None:
            self.symm = symm_workspace
        elif self.N > 1 and algo == K.ALGO_SYMM:
            # fused NVLS collectives: unit buffers and accumulators live in one
            # symmetric allocation; the AG reads the fp32 master directly
            import torch.distributed as dist
            gname = group_name or dist.group.WORLD.group_name
            err = None
            try:
                self.symm = K.SymmWorkspace(self.symm_regions(arch), gname, dev, rank, self.N,
                                            ctas=symm_ctas)
            except Exception as e:            # e.g. no peer mapping on this fabric
                err = f"{type(e).__name__}: {e}"
            # every rank drops the fused route if any rank could not build the workspace
            if self._group.sum_ranks(int(err is not None)) > 0:
                self.symm = None
                self.symm_error = err or "another rank failed to build the symmetric workspace"
        if self.symm is not None:
            self.ubuf = [self.symm["ub0"], self.symm["ub1"]]
            self.rbuf = self.symm["rbuf"]
            self.acc = [self.symm["acc0"], self.symm["acc1"]]
            self.racc = self.symm["racc"]
        # l_i == 1: the backward accumulates units in PAIRS (one launch over both units'
        # gradients, then both reduce-scatters): half the launches, twice the bytes each
        # (decided from the whole plan so every rank issues its collectives in the same order)
        self.pair_units = self.L.blocks >= 2 and all(a.num_microbatches <= 1
                                                     for a in plan.assignments)
        # units per grouped launch: pairs under collectives (each pair's reduce-scatters
        # overlap the next pair's backward); with one rank nothing overlaps, so the whole
        # backward's bf16 -> fp32 scale-cast is one launch (holds 2 B/param of bf16 grads)
        self.acc_group = self.L.blocks if self.N == 1 else 2
        # l_i > 1: microbatches per accumulate launch. A unit's gradients of
        # consecutive microbatches are held (one extra unit of bf16 gradients per
        # held microbatch) and folded into the fp32 accumulator in one pass
        # (het_accumulate_multi): one read and one write of the accumulator per
        # group instead of per microbatch, bit-identical to one pass each
        self.acc_microbatches = 2
        self.bf16_wire = bf16_wire
        # bf16-wire units: the backward's fused ops write each parameter gradient
        # straight into its slot of the symmetric staging buffer gb{u % 2}
        # (hetstep.grad_destinations), so no het_gather_bf16 copy follows
        self.grad_in_place = True
        # N > 1 option: AdamW of each unit's shard on the RS stream right after that
        # unit's reduce-scatter (overlapping the rest of the backward) instead of one
        # pass over the whole shard at the end of the step. Off by default: at N=4 it
        # left the step rate unchanged (GPT-2 5309 vs 5299, Llama 581 vs 580 samples/s)
        # while the overlapped launches ran at 0.49-0.66 of HBM against 0.89-0.90 for
        # the single pass (profiles/r2z/)
        self.overlap_adamw = False
        # Eq. 1 weights of every rank (the bf16-wire reduce-scatter applies them itself)
        self.rank_weights = [a.microbatch / plan.total_batch for a in plan.assignments]
        self._set_routes(self.symm is not None)
        self.route_check = None
        # fused-collective fault check: the sticky barrier status is copied to pinned
        # host memory after every step's collectives (no device sync) and polled at
        # the start of the next step; a timeout raises K.CollectiveFault
        self._watch = K.StatusWatch() if self.symm is not None else None
        if self.symm is not None and check_routes:
            self.route_check = self._check_symm_routes()
            if not self.route_check["ok"]:       # every rank agrees: all-NCCL routes
                self._set_routes(False)
        if self.N > 1 and self.symm is None:
            self.ubuf = [torch.empty(U, dtype=torch.bfloat16, device=dev) for _ in range(2)]
            self.rbuf = torch.empty(E, dtype=torch.bfloat16, device=dev)
            pad_u = (U + 63) // 64 * 64
            self._acc_pair = torch.zeros(2 * pad_u, dtype=torch.float32, device=dev)
            self.acc = [self._acc_pair[:U], self._acc_pair[pad_u:pad_u + U]]
            self.racc = torch.zeros(E, dtype=torch.float32, device=dev)
        self.ag_stream = torch.cuda.Stream(device=dev) if self.cuda else _NoStream()
        self.rs_stream = torch.cuda.Stream(device=dev) if self.cuda else _NoStream()
        self.unit_seg = segment_offsets(arch.unit_layout())
        self.root_seg = segment_offsets(arch.root_layout())
        self.steps = 0
        self.timers = StepTimers()
        self.launches = 0          # owned-kernel launches (hetstep.so), this process
        self.tracer = None         # trace.StepTracer: per-event CUDA timelines when set
        self.keep_last_graph = True  # l_i = 1: keep the last unit's forward graph (no recompute)
        # activation checkpoint offload (schedule sim.py:226-338):
        # unit-boundary checkpoints go to pinned host memory on a D2H stream after the
        # forward uses them and come back one unit ahead of their recompute on an H2D stream
        self.offload = offload_activations and self.cuda
        # "reference": with l_i >= 2 the simulator's full schedule (unit outputs and
        # upstream gradients make PCIe round trips too: O(1) boundary tensors resident);
        # "checkpoints": only the unit-input checkpoints go to host (O(L * l_i) bytes),
        # the l_i in-flight boundary tensors of the current unit stay on the GPU
        # (O(l_i) bytes) so no round trip sits on the critical path
        if offload_schedule not in ("reference", "checkpoints"):
            raise InputError(f"unknown offload schedule {offload_schedule!r}")
        self.offload_schedule = offload_schedule
        # CUDA graph of the whole step (one rank, no offload, no tracer): after
        # `graph_warmup` eager steps the step is captured once and then replayed;
        # the host only copies the tokens in and refreshes AdamW's 7 coefficients
        # (het_adamw_devcoef), so the ~550 launches of a GPT-2 step cost one
        # samples per head chunk (None: the whole microbatch); set for memory-capped
        # ranks so the logits transient stays a small share of the cap
        self.head_chunk: int | None = None
        self.graph = False
        self.graph_warmup = 2
        self._graph = None
        self._capturing = False
        self._coef: torch.Tensor | None = None
        self._epoch_deltas = [0, 0]
        self._graph_launches = 0
        self._eager_steps = 0
        if self.offload:
            self.d2h_stream = torch.cuda.Stream(device=dev)
            self.h2d_stream = torch.cuda.Stream(device=dev)
            # pinned host copies keyed (microbatch k, consumer unit u): "act" = the input
            # checkpoint of unit u, "grad" = the upstream gradient of unit u
            self._host: dict[tuple[str, int, int], torch.Tensor] = {}
            self._off_ev: dict[tuple[str, int, int], torch.cuda.Event] = {}
            # checkpoint prefetch staging (schedule "checkpoints"): two unit slots
            self._pf_slot: list[list[torch.Tensor] | None] = [None, None]
            self._pf_free: list[torch.cuda.Event | None] = [None, None]
            self._last_d2h: torch.cuda.Event | None = None   # most recent offload

    @staticmethod
    def symm_regions(arch: ArchSpec) -> list[tuple[str, int, torch.dtype]]:
        """Regions of the symmetric workspace: double-buffered gathered bf16 units,
        the gathered root, fp32 unit / root accumulators, bf16-wire gradients."""
        U, E = arch.unit_params, arch.root_params
        return [("ub0", U, torch.bfloat16), ("ub1", U, torch.bfloat16),
                ("rbuf", E, torch.bfloat16), ("acc0", U, torch.float32),
                ("acc1", U, torch.float32), ("racc", E, torch.float32),
                ("gb0", U, torch.bfloat16), ("gb1", U, torch.bfloat16)]

    # ------------------------------------------------------------------ routes
    def _set_routes(self, sym: bool) -> None:
        """Per-unit collective routes (fused symmetric kernels vs NCCL ring), fixed by shape."""
        units = range(self.L.blocks + 1)
        self.ag_route = [K.route_collective("ag", self.L.counts[u], self.N, sym) for u in units]
        # a block of an l_i <= 1 plan can take the bf16 wire: routed as "rs16"
        wire_ok = self.bf16_wire and self.pair_units
        self.rs_route = [K.route_collective("rs16" if wire_ok and u < self.L.blocks else "rs",
                                            self.L.counts[u], self.N, sym) for u in units]
        # fused-route kernel policy per unit (hetstep.symm_policy): plain / multicast,
        # pair relay (AG) or helpers (skewed and single-owner units at N >= 3)
        mc = self.symm is not None and self.symm.multicast
        self.ag_policy = [K.symm_policy("ag", self.L.counts[u], self.N, multicast=mc)
                          if self.ag_route[u] == "symm" else None for u in units]
        # a fused RS whose successor (RS order: L-1..0, root) is not fused must end with a
        # cross-rank barrier: nothing later proves that peers finished reading its acc
        order = list(range(self.L.blocks - 1, -1, -1)) + [self.L.root]
        self.rs_end = {u: self.rs_route[u] == "symm" and
                       (i + 1 == len(order) or self.rs_route[order[i + 1]] != "symm")
                       for i, u in enumerate(order)}
        self.need_shadow = not sym or "nccl" in self.ag_route
        # l_i <= 1 on every rank: a fused-route unit's gradient crosses the wire as the
        # unscaled bf16 microbatch gradient; the reduce-scatter applies w_j and the
        # cast (het_symm_reduce_scatter_bf16), half the link bytes of the fp32 form
        self.wire16 = [sym and self.bf16_wire and self.pair_units and u < self.L.blocks and
                       self.rs_route[u] == "symm" for u in units]
        self.rs_policy = [K.symm_policy("rs16" if self.wire16[u] else "rs", self.L.counts[u],
                                        self.N, multicast=mc)
                          if self.rs_route[u] == "symm" else None for u in units]
        # the helper reduce-scatter ends with the cross-rank barrier in-kernel
        for u in units:
            if self.rs_policy[u] in (K.SYMM_HELPERS, K.SYMM_HELPERS_MC):
                self.rs_end[u] = True
        if self.pair_units:
            for u in range(self.L.blocks):
                second = (self.L.blocks - 1 - u) % 2 == 1 or u == 0
                if self.rs_route[u] == "symm" and second:
                    self.rs_end[u] = True   # nothing later proves peers finished reading it

    def _check_symm_routes(self) -> dict:
        """Known-answer check of every fused collective shape this plan uses,
        run once at construction on the real symmetric workspace (the fused
        kernels are specialised per rank count; this proves the specialisation
        for THIS world size before a step trusts it). Exactly representable
        integer patterns make the expected bf16 gather and fp32 sum
        order-independent. Any mismatch or barrier timeout on any rank turns
        every route to NCCL on every rank. Only this rank's stream is
        synchronised (never the device): ranks driven from threads of one
        process (tests/vranks.py) must not wait on each other's spinning kernels."""
        import torch.distributed as dist
        dev = self.device
        shapes = {}
        for u in range(self.L.blocks + 1):
            key = (tuple(self.L.counts[u]), tuple(self.L.offsets[u]))
            shapes.setdefault(key, (u, self.ag_route[u] == "symm", self.rs_route[u] == "symm"))
        K.SymmWorkspace.status(reset=True)
        bad = 0
        checked = 0
        # every rank has finished its construction (allocations, pinned buffers,
        # streams: implicit device synchronisation points) before any rank enters a
        # fused kernel whose barrier waits for it
        self._current().synchronize()
        self.symm.handle.barrier()

        def pattern(idx: torch.Tensor, r: int) -> torch.Tensor:
            return (((idx * 7 + r * 13) % 251) - 125).to(torch.float32)

        for (counts, offsets), (u, ag, rs) in shapes.items():
            size = sum(counts)
            root = u == self.L.root
            ub, acc = ("rbuf", "racc") if root else ("ub0", "acc0")
            lo, cnt = offsets[self.rank], counts[self.rank]
            if ag:
                src = pattern(torch.arange(lo, lo + cnt, device=dev), 0)
                self.symm.allgather_pack(src, ub, 0, counts, offsets, stream=self._current(),
                                         policy=self.ag_policy[u])
                want = pattern(torch.arange(size, device=dev), 0).to(torch.bfloat16)
                bad += int(not torch.equal(self.symm[ub][:size], want))
                checked += 1
            if rs and self.wire16[u]:        # bf16 wire: weights and cast in the RS
                gb = self.symm["gb0"]
                gb[:size].copy_(pattern(torch.arange(size, device=dev), self.rank))
                out = torch.full((cnt,), float("nan"), device=dev)
                self._current().synchronize()
                self.symm.handle.barrier()
                hel = self.rs_policy[u] == K.SYMM_HELPERS
                self.symm.reduce_scatter_bf16("gb0", 0, out, counts, offsets, self.rank_weights,
                                              end_barrier=True, stream=self._current(),
                                              policy=self.rs_policy[u],
                                              stage="acc0" if hel else None)
                idx = torch.arange(lo, lo + cnt, device=dev)
                want = torch.zeros(cnt, device=dev)
                for r, w in enumerate(self.rank_weights):
                    if w != 0.0:
                        want = want + torch.tensor(w, dtype=torch.float32, device=dev) * \
                            pattern(idx, r)
                bad += int(not torch.equal(out, want))
                checked += 1
                gb.zero_()
            if rs:
                self.symm[acc][:size].copy_(pattern(torch.arange(size, device=dev), self.rank))
                out = torch.full((cnt,), float("nan"), device=dev)
                self._current().synchronize()
                self.symm.handle.barrier()
                pol = K.symm_policy("rs", counts, self.N, self.symm.multicast)
                self.symm.reduce_scatter(acc, 0, out, counts, offsets, end_barrier=True,
                                         stream=self._current(), policy=pol)
                idx = torch.arange(lo, lo + cnt, device=dev)
                want = sum(pattern(idx, r) for r in range(self.N))
                bad += int(not torch.equal(out, want))
                checked += 1
        self._current().synchronize()
        status = K.SymmWorkspace.status(reset=True)
        failures = self._group.sum_ranks(bad + (1 if status else 0))
        self.symm.handle.barrier()
        for name in ("ub0", "acc0", "rbuf", "racc", "gb0"):
            self.symm[name].zero_()
        self._current().synchronize()
        self.symm.handle.barrier()
        return {"ok": failures == 0, "checked": checked, "failures": failures, "status": status}

    # ------------------------------------------------------------------ params
    def _local(self, buf: torch.Tensor, u: int) -> torch.Tensor:
        off, cnt = self.L.local_range(u)
        return buf[off:off + cnt]

    def load_full_units(self, units: list[torch.Tensor]) -> None:
        """Install full fp32 unit vectors (L blocks then the root) and take this
        rank's shards; refreshes the bf16 shadow."""
        if len(units) != self.L.blocks + 1:
            raise InputError("need one tensor per block plus the root")
        for u, full in enumerate(units):
            if full.numel() != self.L.unit_size(u):
                raise InputError(f"unit {u}: wrong size")
            o = self.L.offsets[u][self.rank]
            c = self.L.counts[u][self.rank]
            self._local(self.p32, u).copy_(full.reshape(-1)[o:o + c].to(self.device,
                                                                        torch.float32))
        self.refresh_shadow()
        self.m32.zero_()
        self.v32.zero_()
        self.steps = 0

    def refresh_shadow(self) -> None:
        """Re-derive the bf16 all-gather shadow from the fp32 master (kernel 1)."""
        K.pack_bf16(self.p32, self.p16)
        self.launches += 1

    def init_params(self, seed: int = 0) -> None:
        """Deterministic N(0, 0.02) init; every rank derives the same full
        units (seeded per unit) and keeps its own ranges."""
        units = []
        for u in range(self.L.blocks + 1):
            gen = torch.Generator(device=self.device)
            gen.manual_seed(seed * 100003 + u)
            layout = self.arch.root_layout() if u == self.L.root else self.arch.unit_layout()
            units.append(init_flat(layout, gen, self.device))
        self.load_full_units(units)

    # ------------------------------------------------------------------ offload
    def _offload(self, what: str, k: int, u: int, t: torch.Tensor, comp, span_u: int,
                 phase: str) -> None:
        """D2H of `t` (key what/k/u) on the D2H stream once `comp` produced it; the
        GPU copy is released when the copy lands."""
        key = (what, k, u)
        host = self._host.get(key)
        if host is None or host.shape != t.shape:
            host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            self._host[key] = host
        self.d2h_stream.wait_stream(comp)
        kind = "offload_act" if what == "act" else "offload_grad"
        with self._span(kind, span_u, k + 1, phase, self.d2h_stream):
            with torch.cuda.stream(self.d2h_stream):
                host.copy_(t, non_blocking=True)
        t.record_stream(self.d2h_stream)       # GPU copy released once the D2H lands
        ev = torch.cuda.Event()
        ev.record(self.d2h_stream)
        self._off_ev[key] = ev
        self._last_d2h = ev

    def _fetch(self, what: str, k: int, u: int, phase: str):
        """H2D of the host copy what/k/u on the H2D stream (after its D2H landed);
        returns (device tensor, event the consumer waits on)."""
        key = (what, k, u)
        self.h2d_stream.wait_event(self._off_ev[key])
        # the simulator's hand-off (sim.py:226-338): a prefetch lands only after the
        # previous offload drained, so at most two boundary tensors are resident
        # (the reference's 2-item contract, test_acceptance.py:157-186)
        if self._last_d2h is not None:
            self.h2d_stream.wait_event(self._last_d2h)
        kind = "prefetch_act" if what == "act" else "prefetch_grad"
        with self._span(kind, u, k + 1, phase, self.h2d_stream):
            with torch.cuda.stream(self.h2d_stream):
                t = self._host[key].to(self.device, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(self.h2d_stream)
        return t, ev

    def _prefetch_unit(self, u: int, nmb: int) -> tuple[list[torch.Tensor], torch.cuda.Event]:
        """All microbatch inputs of unit u back to the GPU (one unit of look-ahead),
        into one of two persistent staging slots (unit parity) allocated once on
        the compute stream: no per-fetch allocation on the H2D stream, whose
        blocks (freed only once the compute stream passed them) fragmented the
        caching allocator under tight emulated HBM caps into cudaFree retries.
        The H2D copies wait for the slot's previous unit (u + 2) to finish its
        backward."""
        slot = u % 2
        host0 = self._host[("act", 0, u)]
        bufs = self._pf_slot[slot]
        if bufs is None or len(bufs) != nmb or bufs[0].shape != host0.shape:
            bufs = [torch.empty(host0.shape, dtype=host0.dtype, device=self.device)
                    for _ in range(nmb)]
            self._pf_slot[slot] = bufs
            self.h2d_stream.wait_stream(self._current())     # allocated on the compute stream
        if self._pf_free[slot] is not None:
            self.h2d_stream.wait_event(self._pf_free[slot])
        out = []
        for k in range(nmb):
            key = ("act", k, u)
            self.h2d_stream.wait_event(self._off_ev[key])
            with self._span("prefetch_act", u, k + 1, "bwd", self.h2d_stream):
                with torch.cuda.stream(self.h2d_stream), torch.no_grad():
                    bufs[k].copy_(self._host[key], non_blocking=True)
            out.append(bufs[k].detach())
        ev = torch.cuda.Event()
        ev.record(self.h2d_stream)
        return out, ev

    def _take(self, fetched, comp) -> torch.Tensor:
        t, ev = fetched
        comp.wait_event(ev)
        t.record_stream(comp)
        return t

    # ------------------------------------------------------------------ comm
    def _event(self, stream):
        ev = torch.cuda.Event() if self.cuda else _NoStream()
        ev.record(stream)
        return ev

    def _current(self):
        return torch.cuda.current_stream(self.device) if self.cuda else _NoStream()

    def _region(self, t: torch.Tensor) -> str:
        for name, v in self.symm.views.items():
            if v.data_ptr() == t.data_ptr():
                return name
        raise InputError("buffer is not in the symmetric workspace")

    def _span(self, kind: str, u: int, mb: int, phase: str, stream):
        """Trace span (simulator schema: blocks are units 1..L, the root is 0)."""
        if self.tracer is None or not self.cuda:
            return contextlib.nullcontext()
        unit = 0 if u == self.L.root else u + 1
        return self.tracer.span(kind, unit, mb, phase, stream)

    def _ag(self, u: int, dst: torch.Tensor, phase: str = "fwd") -> torch.cuda.Event:
        with self._span("allgather", u, 0, phase, self.ag_stream):
            self._ag_issue(u, dst)
        return self._event(self.ag_stream)

    def _ag_issue(self, u: int, dst: torch.Tensor) -> None:
        if self.ag_route[u] == "symm":   # fused pack + NVLS/peer all-gather from fp32 master
            self.symm.allgather_pack(self._local(self.p32, u), self._region(dst), 0,
                                     self.L.counts[u], self.L.offsets[u], stream=self.ag_stream,
                                     policy=self.ag_policy[u])
            self.launches += 1
        else:
            K.allgather_uneven(self._local(self.p16, u), dst, self.L.counts[u],
                               self.L.offsets[u], self.comm_ag, self.rank,
                               K.ALGO_AUTO if self.algo == K.ALGO_SYMM else self.algo,
                               stream=self.ag_stream)

    def _rs(self, u: int, src: torch.Tensor, after: torch.cuda.Event) -> torch.cuda.Event:
        self.rs_stream.wait_event(after)
        with self._span("reducescatter", u, 0, "bwd", self.rs_stream):
            self._rs_issue(u, src)
        if self.overlap_adamw:
            self._adamw_unit(u)
        return self._event(self.rs_stream)

    def _adamw_unit(self, u: int) -> None:
        """AdamW over unit u's (padded) local range on the RS stream, right behind
        the unit's reduce-scatter: the optimizer of the early-reduced units runs
        under the backward of the later ones instead of as one pass at the end of
        the step. The pads are zero in p, g, m and v and stay zero."""
        lo = self.L.local_off[u]
        hi = self.L.local_off[u + 1] if u + 1 <= self.L.root else self.L.local_len
        if hi <= lo:
            return
        shadow = self.p16[lo:hi] if self.need_shadow else None
        a, b = self.timers.pair("adamw", (30.0 if self.need_shadow else 28.0) * (hi - lo))
        if a is not None:
            a.record(self.rs_stream)
        if self._coef is not None:      # graph capture: coefficients staged per replay
            K.adamw_devcoef(self.p32[lo:hi], self.g32[lo:hi], self.m32[lo:hi],
                            self.v32[lo:hi], shadow, self._coef, stream=self.rs_stream)
        else:
            K.adamw(self.p32[lo:hi], self.g32[lo:hi], self.m32[lo:hi], self.v32[lo:hi],
                    shadow, lr=self.opt.lr, beta1=self.opt.betas[0], beta2=self.opt.betas[1],
                    eps=self.opt.eps, weight_decay=self.opt.weight_decay, step=self.steps + 1,
                    stream=self.rs_stream)
        if b is not None:
            b.record(self.rs_stream)
        self.launches += 1

    def _rs_issue(self, u: int, src: torch.Tensor) -> None:
        if self.wire16[u]:               # bf16 wire: weighting + cast inside the RS
            # helpers stage their fp32 sums in the unit's (unused) fp32 accumulator
            hel = self.rs_policy[u] == K.SYMM_HELPERS
            self.symm.reduce_scatter_bf16(f"gb{u % 2}", 0, self._local(self.g32, u),
                                          self.L.counts[u], self.L.offsets[u], self.rank_weights,
                                          end_barrier=self.rs_end[u], stream=self.rs_stream,
                                          policy=self.rs_policy[u],
                                          stage=f"acc{u % 2}" if hel else None)
            self.launches += 1
        elif self.rs_route[u] == "symm":   # switch/peer reduction straight into the fp32 shard
            self.symm.reduce_scatter(self._region(src), 0, self._local(self.g32, u),
                                     self.L.counts[u], self.L.offsets[u],
                                     end_barrier=self.rs_end[u], stream=self.rs_stream,
                                     policy=self.rs_policy[u])
            self.launches += 1
        else:
            K.reduce_scatter_uneven(src, self._local(self.g32, u), self.L.counts[u],
                                    self.L.offsets[u], self.comm_rs, self.rank,
                                    K.ALGO_AUTO if self.algo == K.ALGO_SYMM else self.algo,
                                    stream=self.rs_stream)

    def _unit_flat(self, u: int) -> torch.Tensor:
        if self.N == 1:
            off = self.L.local_off[u]
            return self.p16[off:off + self.L.unit_size(u)]
        return self.rbuf if u == self.L.root else self.ubuf[u % 2]

    def _zero_acc(self, u: int) -> None:
        K.fill(self._acc(u), 0.0)
        self.launches += 1

    def _acc(self, u: int) -> torch.Tensor:
        if self.N == 1:
            return self._local(self.g32, u)
        return self.racc if u == self.L.root else self.acc[u % 2]

    def _acc_base(self, u: int) -> tuple[torch.Tensor, int]:
        """(tensor, element offset) addressing unit u's accumulator, with one base
        shared by both unit accumulators so a paired launch can cover two units."""
        if self.N == 1:
            return self.g32, self.L.local_off[u]
        a0, a = self.acc[0], self.acc[u % 2]
        off = (a.data_ptr() - a0.data_ptr()) // 4
        span = (self.acc[1].data_ptr() - a0.data_ptr()) // 4 + self.acc[1].numel()
        return a0.as_strided((span,), (1,), a0.storage_offset()), off

    def _grad_dst(self, u: int, params: dict) -> dict:
        """Destinations of unit u's parameter gradients in gb{u % 2} (keyed as
        hetstep.grad_out looks them up), including the adjacent-row groups the
        Llama unit multiplies as one matrix (wq|wk|wv, w1|w3)."""
        gb = self.symm[f"gb{u % 2}"]
        out = {}
        for nm, shape in self.arch.unit_layout():
            t, off = params[nm], self.unit_seg[nm]
            out[(t.data_ptr(), tuple(t.shape))] = gb[off:off + t.numel()].view(shape)
        for group in (("wq", "wk", "wv"), ("w1", "w3")):
            if all(g in params for g in group):
                ts = [params[g] for g in group]
                rows = sum(t.shape[0] for t in ts)
                shape = (rows,) + tuple(ts[0].shape[1:])
                off = self.unit_seg[group[0]]
                n = rows * ts[0].shape[1]
                out[(ts[0].data_ptr(), shape)] = gb[off:off + n].view(shape)
        return out

    def _accumulate_units(self, items, names, seg):
        """One het_accumulate (FIRST) over [(u, grads), ...] of several units; units
        on the bf16 wire are staged unscaled into their bf16 buffer instead (only
        the gradients the backward did not already write there)."""
        w16 = [(u, g) for u, g in items if self.wire16[u]]
        items = [(u, g) for u, g in items if not self.wire16[u]]
        if w16:
            stage = []
            base = self.symm["gb0"].data_ptr()
            for u, grads in w16:
                off = (self.symm[f"gb{u % 2}"].data_ptr() - base) // 2
                stage += [(g, off + seg[nm]) for g, nm in zip(grads, names)
                          if g.data_ptr() != base + 2 * (off + seg[nm])]
        if w16 and stage:
            n16 = sum(g.numel() for g, _ in stage)
            gb = self.symm["gb0"]
            span = (self.symm["gb1"].data_ptr() - gb.data_ptr()) // 2 + self.symm["gb1"].numel()
            a, b = self.timers.pair("gather", n16 * 4.0)
            K.gather_bf16(gb.as_strided((span,), (1,), gb.storage_offset()), stage,
                          events=None if a is None else (a, b))
            self.launches += 1
        if not items:
            return
        base = None
        pairs = []
        n = 0
        for u, grads in items:
            t, off = self._acc_base(u)
            base = t if base is None else base
            pairs += [(g, off + seg[nm]) for g, nm in zip(grads, names)]
            n += sum(g.numel() for g in grads)
        a, b = self.timers.pair("accumulate", n * 6.0)
        K.accumulate(base, pairs, True, self.w, events=None if a is None else (a, b))
        self.launches += 1

    def _accumulate(self, acc, grads, names, seg, first):
        n = sum(g.numel() for g in grads)
        a, b = self.timers.pair("accumulate", n * (6.0 if first else 10.0))
        K.accumulate(acc, [(g, seg[nm]) for g, nm in zip(grads, names)], first, self.w,
                     events=None if a is None else (a, b))
        self.launches += 1

    def _head(self, leaves, head_names, y, targets, racc, loss):
        """Loss and gradients of one microbatch's head (final norm, tied LM head,
        cross-entropy): head parameter gradients accumulated into the root
        accumulator, the weighted loss added to `loss`; returns the gradients
        (last: d loss / d y). With head_chunk set, the head runs over row chunks
        of head_chunk samples, each with its share of the gradient (grad_scale),
        so the [rows, vocab] logits transient shrinks by the chunk count: the
        largest single allocation of a memory-capped rank."""
        arch, m = self.arch, y.shape[0]
        c = self.head_chunk if self.head_chunk and self.head_chunk < m else m
        gy = []
        for j0 in range(0, m, c):
            j1 = min(j0 + c, m)
            yj = y if c == m else y[j0:j1].detach().requires_grad_(True)
            frac = (j1 - j0) / m
            lk, grads = head_value_and_grad(arch, leaves, yj, targets[j0:j1],
                                            [leaves[nm] for nm in head_names] + [yj],
                                            grad_scale=frac)
            self._accumulate(racc, grads[:-1], head_names, self.root_seg, first=False)
            loss += lk.detach() * (self.w * frac)
            gy.append(grads[-1])
            del grads
        return [None] * len(head_names) + [gy[0] if len(gy) == 1 else torch.cat(gy)]

    def _accumulate_mb(self, acc, held, names, seg, first):
        """Layered accumulate of consecutive microbatches' gradients of one unit
        (one launch; a single microbatch goes through het_accumulate)."""
        if len(held) == 1:
            self._accumulate(acc, held[0], names, seg, first)
            return
        n = sum(g.numel() for g in held[0])
        a, b = self.timers.pair("accumulate", n * (2.0 * len(held) + (4.0 if first else 8.0)))
        K.accumulate_multi(acc, held, [seg[nm] for nm in names], first, self.w,
                           events=None if a is None else (a, b))
        self.launches += 1

    # ------------------------------------------------------------------ step
    def step(self, tok: torch.Tensor) -> torch.Tensor:
        """One iteration on this rank's [b_i, seq+1] int32 token block (device).
        Returns this rank's Eq. 1-weighted loss contribution sum_k (m_i/B) loss_k
        (a device scalar; the global loss is its sum over ranks)."""
        if self.graph and self.graph_eligible():
            return self._graph_step(tok)
        self._eager_steps += 1
        return self._step(tok)

    def graph_eligible(self) -> bool:
        """No offload, no tracer, a non-idle rank. With several ranks every unit
        must route through the fused collectives, which take their barrier
        epochs from device memory inside a replay (no host counter); ranks
        decide independently, a replaying rank issuing the same epoch sequence
        as an eager one. NCCL-routed units are not captured: steps with NCCL
        graph nodes hung when some ranks ran eagerly (BERT-large N=4, offloading
        ranks eager) and in an all-NCCL N=2 step (profiles/r2z/, r2b4/). N <= 4:
        N=8 never ran on real GPUs here."""
        multi_ok = self.N == 1 or (self.symm is not None and self.N <= 4
                                   and all(r == "symm" for r in self.ag_route)
                                   and all(r == "symm" for r in self.rs_route))
        return (self.cuda and multi_ok and not self.offload and self.tracer is None
                and self.m > 0)

    @property
    def graph_active(self) -> bool:
        return self._graph is not None

    def _graph_step(self, tok: torch.Tensor) -> torch.Tensor:
        if self._graph is None and self._eager_steps < self.graph_warmup:
            self._eager_steps += 1
            return self._step(tok)
        if self._graph is None:
            self._capture(tok)
        if self._watch is not None:
            self._watch.poll()           # earlier replays' collectives: raise on a timeout
        self._g_tok.copy_(tok, non_blocking=True)
        self._stage_coef()
        self._graph.replay()
        self.steps += 1
        if self.symm is not None:
            self.symm.advance_host(self._epoch_deltas)
        if self.N > 1:
            if self._watch is not None:
                self._watch.record(self._current(), f"step {self.steps} on rank {self.rank}")
        K.LAUNCHES += self._graph_launches
        self.launches += self._graph_own
        return self._g_loss.clone()

    def release_graph(self) -> None:
        """Drop the captured step (before the communicators its NCCL nodes use are
        destroyed); the next step runs eagerly and may capture again."""
        if self._graph is not None:
            torch.cuda.synchronize(self.device)
            self._graph = None
            self._eager_steps = 0

    def _stage_coef(self) -> None:
        """AdamW coefficients of the coming step into the device buffer the graph's
        het_adamw_devcoef reads: host math (het_adamw_coef, as het_adamw), a pinned
        slot per step from a small ring (an event guards each slot's reuse), and
        an async H2D copy stream-ordered before the replay."""
        k = self.steps % len(self._coef_pin)
        self._coef_ev[k].synchronize()
        c = K.adamw_coef(lr=self.opt.lr, beta1=self.opt.betas[0], beta2=self.opt.betas[1],
                         eps=self.opt.eps, weight_decay=self.opt.weight_decay,
                         step=self.steps + 1)
        self._coef_pin[k].copy_(torch.tensor(c, dtype=torch.float32))
        self._coef_dev.copy_(self._coef_pin[k], non_blocking=True)
        self._coef_ev[k].record()

    def _capture(self, tok: torch.Tensor) -> None:
        self._g_tok = torch.empty_like(tok)
        self._g_tok.copy_(tok)
        self._coef_dev = torch.zeros(7, dtype=torch.float32, device=self.device)
        self._coef_pin = [torch.zeros(7, dtype=torch.float32).pin_memory() for _ in range(4)]
        self._coef_ev = [torch.cuda.Event() for _ in range(4)]
        for ev in self._coef_ev:
            ev.record()
        cur = self._current()
        # a green-context rank captures on its own compute stream, so the kernel
        # nodes keep the SM partition (torch's default capture stream would not)
        cap_stream = None if cur == torch.cuda.default_stream(self.device) else cur
        if self.symm is not None:       # barrier epochs from device memory from now on
            self.symm.begin_device_epochs(cur)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        timers_on = self.timers.enabled
        if timers_on:           # the replays re-record these (external) events
            self.timers.reset()
            self.timers.external = True
        n0, s0, l0 = K.LAUNCHES, self.steps, self.launches
        self._capturing = True
        try:
            with torch.cuda.graph(g, stream=cap_stream):
                self._g_loss = self._step(self._g_tok, coef=self._coef_dev)
                if self.symm is not None:
                    # the capture stream has joined every AG / RS launch of the step
                    self._epoch_deltas = self.symm.end_device_epochs(self._current())
        finally:
            self.timers.external = False
            self._capturing = False
            if self.symm is not None and self.symm._dev_epoch0 is not None:   # failed capture
                self.symm.epoch = list(self.symm._dev_epoch0)
                self.symm._dev_epoch0 = None
        # the capture issued no work: every replay counts the captured launches
        self._graph_launches = K.LAUNCHES - n0
        self._graph_own = self.launches - l0
        K.LAUNCHES, self.steps, self.launches = n0, s0, l0
        self._graph = g

    def _step(self, tok: torch.Tensor, coef: torch.Tensor | None = None) -> torch.Tensor:
        arch, L, comp = self.arch, self.L, self._current()
        nb, root = L.blocks, L.root
        if self.m > 0 and (tok.shape[0] != self.m * self.l or tok.shape[1] != arch.seq + 1):
            raise InputError(f"rank {self.rank} expects tokens [{self.m * self.l}, {arch.seq + 1}]")
        multi = self.N > 1
        self._coef = coef                # graph capture: AdamW coefficients on the device
        if self._watch is not None and not self._capturing:
            self._watch.poll()           # earlier steps' collectives: raise on a timeout
        unit_names = [nm for nm, _ in arch.unit_layout()]
        root_names = [nm for nm, _ in arch.root_layout()]
        loss = torch.zeros((), dtype=torch.float32, device=self.device)
        if self.tracer is not None and self.cuda:
            self.tracer.begin(comp)

        # ---- forward (+ head) ----------------------------------------------
        # Offload (sim.py:226-338): every unit input checkpoint goes to pinned host memory
        # once its forward consumed it and comes back for its recompute. With l_i >= 2
        # ("deep") the reference schedule is followed in full: unit outputs go to host as
        # soon as they are produced and the next forward microbatch's input is prefetched,
        # upstream gradients likewise in the backward, so O(1) boundary tensors stay on
        # the GPU instead of O(l_i). With l_i = 1 the one in-flight tensor is consumed
        # next, so a round trip would only sit on the critical path.
        ag_ev: dict[int, torch.cuda.Event] = {}
        done_ev: dict[int, torch.cuda.Event] = {}
        if multi:
            self.ag_stream.wait_stream(comp)      # previous step's AdamW wrote p16
            ag_ev[root] = self._ag(root, self.rbuf)
            ag_ev[0] = self._ag(0, self.ubuf[0])
        racc = self._acc(root)
        if multi and not self._capturing:
            # racc no longer read by last step's RS (graph replays are serialised on
            # the launch stream, so a captured step needs no such edge)
            comp.wait_stream(self.rs_stream)
        K.fill(racc, 0.0)
        self.launches += 1

        active = self.m > 0
        mb = [(tok[k * self.m:(k + 1) * self.m, :-1], tok[k * self.m:(k + 1) * self.m, 1:])
              for k in range(self.l)] if active else []
        nmb = len(mb)
        off = self.offload and nmb > 0
        deep = off and nmb >= 2 and self.offload_schedule == "reference"
        # one microbatch, no offload: the last unit's forward runs with autograd and its
        # graph is kept for the backward, which follows right after the head (its
        # recompute would redo exactly that forward)
        keep_last = self.keep_last_graph and nmb == 1 and not off
        kept = None
        h: list[list[torch.Tensor | None]] = [[None] * (nb + 1) for _ in mb]
        dy: list[torch.Tensor | None] = [None] * nmb
        fetched: dict[tuple[str, int, int], tuple] = {}
        if multi:
            comp.wait_event(ag_ev[root])
        rp = views(self._unit_flat(root), arch.root_layout())
        leaves = {nm: t.requires_grad_(True) for nm, t in
                  views(self._unit_flat(root), arch.root_layout()).items()}
        head_names = [nm for nm in root_names if nm != "wpe"]
        with torch.no_grad():
            for u in range(nb):
                if multi:
                    if u + 1 < nb:
                        if u >= 1:
                            self.ag_stream.wait_event(done_ev[u - 1])
                        ag_ev[u + 1] = self._ag(u + 1, self.ubuf[(u + 1) % 2])
                    comp.wait_event(ag_ev[u])
                p = views(self._unit_flat(u), arch.unit_layout())
                for k in range(nmb):
                    if u == 0:
                        with self._span("fwd_compute", root, k + 1, "fwd", comp):
                            x = embed_forward(arch, rp, mb[k][0])
                    elif deep:
                        x = self._take(fetched.pop(("act", k, u)), comp)
                    else:
                        x = h[k][u]
                    if deep:                      # next forward microbatch's input
                        nk, nu = (k + 1, u) if k + 1 < nmb else (0, u + 1)
                        if 1 <= nu < nb:
                            fetched[("act", nk, nu)] = self._fetch("act", nk, nu, "fwd")
                    if keep_last and u == nb - 1:
                        pk = {nm: t.requires_grad_(True) for nm, t in
                              views(self._unit_flat(u), arch.unit_layout()).items()}
                        with self._span("fwd_compute", u, k + 1, "fwd", comp):
                            x = x.requires_grad_(True)
                            with torch.enable_grad():
                                y = block_forward(arch, pk, x)
                        kept = (x, y, [pk[nm] for nm in unit_names])
                    else:
                        with self._span("fwd_compute", u, k + 1, "fwd", comp):
                            y = block_forward(arch, p, x)
                    if off and (u == 0 or not deep):
                        self._offload("act", k, u, x, comp, u, "fwd")   # recompute input
                    h[k][u] = None if off else x
                    if deep and u + 1 < nb:
                        self._offload("act", k, u + 1, y, comp, u, "fwd")
                        y = None
                    if u + 1 < nb:
                        h[k][u + 1] = y
                        continue
                    # head + loss of microbatch k right behind the last unit's forward
                    with self._span("head", root, k + 1, "fwd", comp):
                        if not y.requires_grad:
                            y.requires_grad_(True)
                        grads = self._head(leaves, head_names, y, mb[k][1], racc, loss)
                    if deep:
                        self._offload("grad", k, nb - 1, grads[-1], comp, nb, "bwd")
                    else:
                        dy[k] = grads[-1]
                    del grads, y
                done_ev[u] = self._event(comp)
        pref: dict[int, tuple[list[torch.Tensor], torch.cuda.Event]] = {}
        if deep:                                  # turnaround (sim.py:270-274)
            fetched[("act", 0, nb - 1)] = self._fetch("act", 0, nb - 1, "bwd")
            fetched[("grad", 0, nb - 1)] = self._fetch("grad", 0, nb - 1, "bwd")
        elif off:
            pref[nb - 1] = self._prefetch_unit(nb - 1, nmb)

        # ---- backward --------------------------------------------------------
        rs_ev: dict[int, torch.cuda.Event] = {}
        pending: list[tuple[int, list[torch.Tensor]]] = []     # paired-accumulate queue
        wpe_off = self.root_seg.get("wpe") if arch.kind != "llama" else None
        for u in reversed(range(nb)):
            if multi:
                # prefetch u-1 unless it is still resident from the forward
                if u - 1 >= 0 and u - 1 < nb - 2:
                    self.ag_stream.wait_event(done_ev[u + 1])
                    ag_ev[u - 1] = self._ag(u - 1, self.ubuf[(u - 1) % 2], "bwd")
                if u < nb - 2:
                    comp.wait_event(ag_ev[u])
            # acc[u % 2] is rewritten by this unit's first accumulate: its last readers
            # are RS(u+2) on this rank and, through the fused RS, on every peer (my
            # RS(u+1) having passed its start barrier proves every rank finished
            # RS(u+2)). The waits sit right before that first accumulate, so the
            # reduce-scatters overlap this unit's recompute and backward.
            acc_free = [rs_ev[v] for v in (u + 2, u + 1) if multi and not self.pair_units
                        and v in rs_ev and (v == u + 2 or self.symm is not None)]
            if off and not deep:
                if u - 1 >= 0:                    # one unit of look-ahead
                    pref[u - 1] = self._prefetch_unit(u - 1, nmb)
                tensors, ev = pref.pop(u)
                comp.wait_event(ev)
                for k, t in enumerate(tensors):
                    h[k][u] = t
            acc = self._acc(u)
            held: list[list[torch.Tensor]] = []      # microbatch gradients awaiting accumulate
            flat = self._unit_flat(u)
            pl = {nm: t.requires_grad_(True) for nm, t in views(flat, arch.unit_layout()).items()}
            plist = [pl[nm] for nm in unit_names]
            in_place = (self.grad_in_place and self.pair_units and self.wire16[u] and nmb > 0
                        and self.cuda)
            if in_place:
                # the backward writes gb{u % 2} itself: its last readers are RS(u+2) here
                # and on every peer; RS(u+1) / RS(u+2), whichever is issued and carries
                # the end barrier, proves they finished
                for w_ in (u + 1, u + 2):
                    if w_ in rs_ev:
                        comp.wait_event(rs_ev[w_])
                dst = K.grad_destinations(self._grad_dst(u, pl))
            else:
                dst = contextlib.nullcontext()
            for k in range(nmb):
                nk, nu = (k + 1, u) if k + 1 < nmb else (0, u - 1)
                if deep:
                    x = self._take(fetched.pop(("act", k, u)), comp)
                    if nu >= 0:                   # next recompute input (at RA start)
                        fetched[("act", nk, nu)] = self._fetch("act", nk, nu, "bwd")
                else:
                    x = h[k][u]
                if kept is not None and u == nb - 1:
                    x, y, plist_u = kept             # graph kept from the forward
                    kept = None
                else:
                    plist_u = plist
                    with self._span("recompute", u, k + 1, "bwd", comp):
                        x = x.requires_grad_(True)
                        with torch.enable_grad():
                            y = block_forward(arch, pl, x)
                if deep:
                    g_in = self._take(fetched.pop(("grad", k, u)), comp)
                    if nu >= 0:                   # next upstream gradient (at B start)
                        fetched[("grad", nk, nu)] = self._fetch("grad", nk, nu, "bwd")
                else:
                    g_in = dy[k]
                with self._span("bwd_compute", u, k + 1, "bwd", comp), dst:
                    grads = torch.autograd.grad(y, plist_u + [x], g_in)
                    h[k][u] = dy[k] = None
                    if self.pair_units:
                        unit_grads = list(grads[:-1])
                    else:
                        held.append(list(grads[:-1]))
                        if len(held) >= self.acc_microbatches or k == nmb - 1:
                            for ev_ in acc_free:
                                comp.wait_event(ev_)
                            acc_free = []
                            self._accumulate_mb(acc, held, unit_names, self.unit_seg,
                                                first=(k + 1 == len(held)))
                            held = []
                if u == 0:
                    # fused embedding backward: token / position rows summed in fp32 straight
                    # into the root accumulator (no dense [vocab, d] bf16 gradient,
                    # deterministic order)
                    with self._span("embed_bwd", root, k + 1, "bwd", comp):
                        K.embedding_grad(racc, self.root_seg["wte"], wpe_off, grads[-1],
                                         mb[k][0], arch.seq, self.w)
                        self.launches += 1
                elif deep:
                    self._offload("grad", k, u - 1, grads[-1], comp, u, "bwd")
                else:
                    dy[k] = grads[-1]
                del grads, y, x, g_in
            if multi and nmb == 0 and not self.wire16[u]:
                # an idle rank contributes zeros; its acc may hold a helper
                # reduce-scatter's staged sums from the last use of this buffer
                for ev_ in acc_free:
                    comp.wait_event(ev_)
                acc_free = []
                self._zero_acc(u)
            done_ev[u] = self._event(comp)
            if off and not deep:
                self._pf_free[u % 2] = done_ev[u]    # staging slot of unit u reusable
            if not self.pair_units:
                if multi:
                    rs_ev[u] = self._rs(u, acc, done_ev[u])
                continue
            pending.append((u, unit_grads if mb else []))   # idle ranks still reduce-scatter
            if len(pending) < self.acc_group and u > 0:
                continue                             # wait for the group's last unit
            if multi:
                # the group's accumulators are rewritten: their previous readers are
                # RS(v+2) here and on every peer. RS(v+1), when issued already, is the
                # later one; with an odd block count the last group is unit 0 alone,
                # and RS(2) (first of its pair, no end barrier) proves only this
                # rank's read, so RS(1) (end barrier) must be waited on too
                for v, _ in pending:
                    for w_ in (v + 2, v + 1):
                        if w_ in rs_ev:
                            comp.wait_event(rs_ev[w_])
            if mb:
                self._accumulate_units([p for p in pending if p[1]], unit_names, self.unit_seg)
            elif multi:              # idle rank: zeros (helpers may have staged sums there)
                for v, _ in pending:
                    if not self.wire16[v]:
                        self._zero_acc(v)
            ev = self._event(comp)
            if multi:
                for v, _ in pending:
                    rs_ev[v] = self._rs(v, self._acc(v), ev)
            pending = []

        # ---- root RS -----------------------------------------------------------
        if multi:
            rs_ev[root] = self._rs(root, racc, self._event(comp))
            comp.wait_event(rs_ev[root])            # RS stream is in order: all shards ready
            if self._watch is not None and not self._capturing:   # replays: _graph_step
                self._watch.record(comp, f"step {self.steps + 1} on rank {self.rank}")

        # ---- optimizer -------------------------------------------------------
        self.steps += 1
        if multi and self.overlap_adamw:       # already applied unit by unit (_adamw_unit)
            return loss
        a, b = self.timers.pair("adamw", (30.0 if self.need_shadow else 28.0) *
                                self.L.local_len)
        if a is not None:
            a.record()
        shadow = self.p16 if self.need_shadow else None   # fused AG reads p32 itself
        with self._span("optimizer", root, 0, "opt", comp):
            if coef is not None:        # graph capture: coefficients staged per replay
                K.adamw_devcoef(self.p32, self.g32, self.m32, self.v32, shadow, coef)
            else:
                K.adamw(self.p32, self.g32, self.m32, self.v32, shadow, lr=self.opt.lr,
                        beta1=self.opt.betas[0], beta2=self.opt.betas[1], eps=self.opt.eps,
                        weight_decay=self.opt.weight_decay, step=self.steps)
        if b is not None:
            b.record()
        self.launches += 1
        return loss

    def check_faults(self) -> None:
        """Wait for every step issued so far and raise K.CollectiveFault if any
        fused collective's cross-rank barrier timed out (its outputs are invalid)."""
        if self._watch is not None:
            self._watch.check()

    # ------------------------------------------------------------------ views for tests
    def full_units(self, which: str = "p32") -> list[torch.Tensor]:
        """All-gather the full fp32 vectors of `which` (p32/g32/m32/v32) for
        every unit (test/debug helper; a collective on multi-rank)."""
        src = getattr(self, which)
        out = []
        for u in range(self.L.blocks + 1):
            full = torch.empty(self.L.unit_size(u), dtype=torch.float32, device=self.device)
            K.allgather_uneven(self._local(src, u).contiguous(), full, self.L.counts[u],
                               self.L.offsets[u], self.comm_ag, self.rank)
            out.append(full)
        return out
