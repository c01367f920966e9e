#!/usr/bin/env python
"""Benchmark of the uneven-FSDP train step (BASELINE.json metric: train
samples/s at 1/2/4/8 B200, emulated heterogeneous; uneven AG/RS bus GB/s in
bench_collectives.py).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config gpt2_small]
  torchrun --nproc-per-node N ... bench.py --gpus N ...     (one rank per GPU)
  python bench.py --impl reference ...                      (CPU reference arm)

A step = one full Cephalo iteration (AG, layered fwd/bwd, weighted RS,
AdamW) of the named config on N GPUs with global batch batch_per_gpu * N
(weak scaling). Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import contextlib
import gc
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2411_01075_b200 import hetstep as K  # noqa: E402
from paper_2411_01075_b200.configs import CONFIGS, build_job  # noqa: E402
from paper_2411_01075_b200.data import rank_tokens  # noqa: E402
from paper_2411_01075_b200.emulate import emulate_tier  # noqa: E402
from paper_2411_01075_b200.step import AdamWConfig, UnevenFSDPTrainer  # noqa: E402

SEED = 1234
OPT = AdamWConfig()
HBM_FALLBACK = 6650.0


def peaks() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return HBM_FALLBACK, "fallback"


def bf16_sustained() -> float:
    """Sustained dense bf16 TFLOP/s from MEASURED_PEAKS.json (B200_PROFILING.md
    fallback otherwise)."""
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["bf16_tflops_sustained"])
    except Exception:
        return 1388.5


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled while the timed
    region runs: NVML every 50 ms (nvidia-smi every 200 ms if NVML is absent),
    in a separate PROCESS, so the sampler never takes the launching thread's
    GIL (a sampler thread measurably slowed launch-heavy steps)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits, in the order of the query above
    BITS = (0x8, 0x40, 0x20, 0x4)
    # the sampler process: initialises NVML, prints "ready", waits for a "go" line,
    # then prints one CSV row per sample until stdin closes
    SCRIPT = r"""
import subprocess, sys, threading
idx, q, bits = int(sys.argv[1]), sys.argv[2], [int(b) for b in sys.argv[3].split(",")]
try:
    import pynvml as nv
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(idx)
except Exception:
    nv = None
print("ready", flush=True)
sys.stdin.readline()
stop = threading.Event()
threading.Thread(target=lambda: (sys.stdin.read(), stop.set()), daemon=True).start()
while not stop.is_set():
    try:
        if nv is not None:
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            row = [str(sm), str(mx)] + ["Active" if rs & b else "Not Active" for b in bits]
        else:
            out = subprocess.run(["nvidia-smi", "-i", str(idx), "--query-gpu=" + q,
                                  "--format=csv,noheader,nounits"], capture_output=True,
                                 text=True, timeout=5).stdout.strip()
            row = [x.strip() for x in out.split(",")] if out else None
        if row:
            print(",".join(row), flush=True)
    except Exception:
        pass
    stop.wait(0.05 if nv is not None else 0.2)
"""

    def __init__(self, index: int):
        """Starts the sampler process (and its NVML init) now, well before the
        timed region; sampling begins at __enter__."""
        self.index, self.rows, self._p = index, [], None
        try:
            self._p = subprocess.Popen(
                [sys.executable, "-c", self.SCRIPT, str(self.index), self.Q,
                 ",".join(str(b) for b in self.BITS)],
                stdin=subprocess.PIPE, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
        except Exception:
            self._p = None

    def __enter__(self):
        if self._p is not None:
            try:
                self._p.stdout.readline()       # "ready"
                self._p.stdin.write("go\n")
                self._p.stdin.flush()
            except Exception:
                self._p = None
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        try:
            out, _ = self._p.communicate(input="", timeout=10)
        except Exception:
            self._p.kill()
            out = ""
        self.rows = [line.split(",") for line in out.splitlines() if "," in line]

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def traffic_from_profile(kernel: str, algo_bytes: float):
    """DRAM bytes per launch of the kernel from the committed ncu --set full
    summary (profiles/ncu_summary.json), or None when not captured."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())[f"het_{kernel}"]
        return {"dram_bytes_per_launch": d["dram_bytes"], "config": d.get("config"),
                "ratio_to_algorithmic_at_capture": d["dram_bytes"] / d["algorithmic_bytes"]}
    except Exception:
        return None


def setup_dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def make_comms(world: int, rank: int):
    if world == 1:
        return None, None
    ids = [K.unique_id(), K.unique_id()] if rank == 0 else [None, None]
    dist.broadcast_object_list(ids, src=0)
    return K.Comm(ids[0], world, rank), K.Comm(ids[1], world, rank)


def cpu_reference_rate(config: str, global_batch: int, max_seconds: float = 20.0,
                       steps: int | None = None, warmup: int = 1) -> dict:
    """The oracle step (torch CPU fp32; oracle/model_oracle.py) timed on this
    host's cores on a bounded sample of the workload, amortised like the GPU
    step: each timed CPU step runs the forward + backward of ONE sample
    (Eq. 1-weighted, as one rank of the step) and one AdamW over the whole
    model; the rate of a global_batch-sample step is then
        B / (B * t_sample + t_adamw),
    the per-sample and per-step parts measured separately. No planner call and
    nothing from the package's native libraries: the workload comes from the
    config's architecture and batch alone."""
    from oracle import model_oracle as MO
    from paper_2411_01075_b200.data import tokens
    from paper_2411_01075_b200.model import ARCHS, init_flat
    cores = len(os.sched_getaffinity(0))
    torch.set_num_threads(cores)
    arch = ARCHS[CONFIGS[config].arch]
    units = []
    for u in range(arch.layers + 1):
        g = torch.Generator().manual_seed(u)
        units.append(init_flat(arch.root_layout() if u == arch.layers else arch.unit_layout(), g,
                               "cpu"))
    opt = dict(lr=OPT.lr, beta1=OPT.betas[0], beta2=OPT.betas[1], eps=OPT.eps,
               weight_decay=OPT.weight_decay)
    params = units[:-1] + [units[-1]]
    mom = [(torch.zeros_like(t), torch.zeros_like(t)) for t in params]

    def one(n: int) -> tuple[float, float]:
        tok = tokens(np.array([n % global_batch]), arch.seq, arch.vocab, SEED, n)
        t0 = time.perf_counter()
        gu, gr, _ = MO.weighted_gradient(arch, units[:-1], units[-1], [tok],
                                         [(1, 1)])
        t1 = time.perf_counter()
        with torch.no_grad():
            for t, g, (m, v) in zip(params, gu + [gr], mom):
                MO.adamw_(t, g, m, v, n + 1, **opt)
        return t1 - t0, time.perf_counter() - t1

    for w in range(warmup):
        one(10_000 + w)
    fb, ad, n = [], [], 0
    while True:
        a, b = one(n)
        fb.append(a)
        ad.append(b)
        n += 1
        if (steps is not None and n >= steps) or (steps is None and sum(fb) + sum(ad) >= max_seconds):
            break
    t_sample, t_adamw = float(np.mean(fb)), float(np.mean(ad))
    rate = global_batch / (global_batch * t_sample + t_adamw)
    return {"value": rate, "unit": "samples/s", "cores": cores, "kind": "port",
            "sample": f"{n} timed CPU steps (after {warmup} warm-up), each = forward+backward of "
                      f"1 sample of {config} (seq {arch.seq}) + one AdamW over all "
                      f"{arch.layers * arch.unit_params + arch.root_params} params, torch CPU "
                      f"fp32 oracle (oracle/model_oracle.py); rate of the {global_batch}-sample "
                      f"step = B / (B * {t_sample * 1e3:.1f} ms + {t_adamw * 1e3:.1f} ms)",
            "sample_ms": t_sample * 1e3, "adamw_ms": t_adamw * 1e3,
            "seconds": float(sum(fb) + sum(ad))}


def describe(config: str, world: int) -> str:
    """The workload as run at this rank count (tiers: configs.CONFIGS)."""
    from collections import Counter
    cfg = CONFIGS[config]
    tiers = [cfg.tiers[i % len(cfg.tiers)] for i in range(world)]
    tally = ", ".join(f"{k} x{v}" for k, v in Counter(tiers).items())
    if world == 1:
        return (f"{cfg.description}; N=1 runs the first tier alone ({tiers[0]}), "
                f"the uneven split starts at N=2")
    return f"{cfg.description}; N={world} tiers: {tally}"


def run_reference(args) -> None:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = max(args.gpus, world)
    cfg = CONFIGS[args.config]
    from paper_2411_01075_b200.model import ARCHS
    B = cfg.batch_per_gpu * n               # the GPU arm's global batch (weak scaling)
    ref = cpu_reference_rate(args.config, B, steps=args.steps, warmup=args.warmup)
    line = {"metric": "train samples/s", "value": ref["value"], "unit": "samples/s",
            "impl": "reference", "n_gpus": n, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "dtype": "f32",
            "data": "synthetic", "scaling": "weak",
            "config": {"workload": args.config, "description": describe(args.config, n),
                       "global_batch": B, "seq_len": ARCHS[cfg.arch].seq},
            "cpu_baseline": {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": ref["value"], "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def tier_capacity(job, no_emulate: bool) -> float:
    from paper_2411_01075_b200.configs import TIERS
    if no_emulate:
        return float(len(job.cluster.gpus))
    return float(sum(TIERS[g.profile_key][0] for g in job.cluster.gpus))


def route_summary(tr) -> dict | str:
    """Which collective route each unit took and the fused kernels' startup
    known-answer check (step._check_symm_routes)."""
    if tr.N == 1:
        return "none"
    return {"ag": {r: tr.ag_route.count(r) for r in sorted(set(tr.ag_route))},
            "rs": {r: tr.rs_route.count(r) for r in sorted(set(tr.rs_route))},
            "ag_relay_units": sum(1 for p in getattr(tr, "ag_policy", []) if p == 3),
            "symm_self_check": tr.route_check, "symm_error": tr.symm_error,
            "rs_bf16_wire_units": sum(tr.wire16)}

def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="gpt2_small", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--trace-dir", default=None,
                    help="also trace one extra step per rank (CUDA events) and write "
                         "rank<i>.jsonl / rank<i>.chrome.json / lint + per-layer report there")
    ap.add_argument("--analytic-profiles", action="store_true",
                    help="plan from the analytic tier profiles instead of the B200-measured ones "
                         "(paper_2411_01075_b200/profiles_b200/)")
    ap.add_argument("--no-emulate", action="store_true",
                    help="run every rank on the full B200 (no green-context SM partition or "
                         "memory cap from the cluster spec)")
    ap.add_argument("--offload", default="auto", choices=["auto", "on", "off"],
                    help="activation-checkpoint offload to pinned host memory; auto = on "
                         "for ranks the plan gives l_i > 1 (layered GA, PAPER.md:388-392)")
    ap.add_argument("--offload-schedule", default="checkpoints",
                    choices=["checkpoints", "reference"],
                    help="checkpoints: only unit-input checkpoints make the host round trip; "
                         "reference: the simulator's full schedule (sim.py:226-338)")
    ap.add_argument("--no-kernel-timers", action="store_true",
                    help="no per-launch CUDA events around the owned kernels in the timed "
                         "region (no roofline line)")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay the step as one CUDA graph (auto: on where eligible: "
                         "one rank, no activation offload)")
    ap.add_argument("--acc-grid", type=int, default=None, choices=[0, 1],
                    help="accumulate grids: 0 persistent (one resident wave), 1 one CTA per "
                         "chunk (library default when unset)")
    ap.add_argument("--adamw-overlap", default="auto", choices=["auto", "on", "off"],
                    help="N>1: AdamW of each unit's shard on the RS stream behind its "
                         "reduce-scatter (on) or one pass over the shard at the end (off)")
    ap.add_argument("--symm-ctas", type=int, default=32,
                    help="CTAs per fused collective launch (each holds one SM while it runs; "
                         "32 measured best in the N=4 steps: profiles/r2c2/)")
    ap.add_argument("--algo", type=int, default=K.ALGO_SYMM,
                    help="collective route for N>1: 4 = fused symmetric-memory kernels "
                         "(default), 0 = NCCL auto, 1 = NCCL send/recv, 2 = NCCL per-owner")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return

    world, rank, local = setup_dist()
    # rank 0's clock sampler process starts (and initialises NVML) now, long
    # before the timed region it samples
    sampler = ClockSampler(local) if rank == 0 else None
    dev = torch.device("cuda", local)
    job = build_job(args.config, world, measured=not args.analytic_profiles)
    comm_ag, comm_rs = make_comms(world, rank)
    # heterogeneity emulation: this rank's tier -> HBM cap + green-context SM partition
    emu = emulate_tier(job.cluster, rank, dev, sm_partition=not args.no_emulate,
                       memory_cap=not args.no_emulate)
    compute_stream = emu.stream if emu.stream is not None else torch.cuda.current_stream()
    ctx = torch.cuda.stream(compute_stream)
    ctx.__enter__()
    layered = job.plan.assignments[rank].num_microbatches > 1
    offload = args.offload == "on" or (args.offload == "auto" and layered)
    tr = UnevenFSDPTrainer(job.arch, job.plan, rank, comm_ag=comm_ag, comm_rs=comm_rs, opt=OPT,
                           device=dev, algo=args.algo if world > 1 else K.ALGO_AUTO,
                           offload_activations=offload,
                           offload_schedule=args.offload_schedule, symm_ctas=args.symm_ctas)
    if args.acc_grid is not None:
        K.set_acc_grid(args.acc_grid)
    if args.adamw_overlap != "auto":
        tr.overlap_adamw = world > 1 and args.adamw_overlap == "on"
    tr.init_params(seed=0)
    # a memory-capped rank runs its head in row chunks so the [rows, vocab]
    # logits transient stays within 10% of its emulated HBM
    logit_bytes = job.arch.seq * job.arch.vocab * 2
    if job.plan.assignments[rank].microbatch * logit_bytes > 0.1 * emu.memory_cap_bytes:
        tr.head_chunk = max(1, int(0.1 * emu.memory_cap_bytes // logit_bytes))
    torch.cuda.empty_cache()     # the full-model init temporaries, before the capped steps
    tr.graph = args.graph != "off" and tr.graph_eligible()
    if args.graph == "on" and not tr.graph:
        raise SystemExit("--graph on: the step is not graph-eligible here (offload, an idle "
                         "rank, no symmetric workspace at N>1, or N>4)")
    arch, plan = job.arch, job.plan
    nsteps = args.warmup + args.steps
    host = [torch.from_numpy(rank_tokens(plan, rank, arch.seq, arch.vocab, SEED, s)).pin_memory()
            for s in range(nsteps)]
    resident = [h.to(dev) for h in host]

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    # ---- device-resident timing (value) ------------------------------------
    # graph mode: the owned-kernel timers are captured with the step (external
    # events the replays re-record), so they are on before the warm-up capture and
    # the summary below reads the last timed replay
    tr.timers.enabled = tr.graph
    for s in range(args.warmup):
        tr.step(resident[s])
    barrier()
    # under a tight emulated HBM cap the caching allocator can still be
    # reshuffling its segments (each "alloc retry" frees its cache and
    # synchronises): keep warming up, at most 12 more steps, until one step
    # runs with no retry on any rank
    extra_warmup = 0
    while extra_warmup < 12:
        r0 = torch.cuda.memory_stats(dev).get("num_alloc_retries", 0)
        tr.step(resident[(args.warmup + extra_warmup) % len(resident)])
        extra_warmup += 1
        barrier()
        if max_over_ranks(float(torch.cuda.memory_stats(dev).get("num_alloc_retries", 0)
                                - r0)) == 0:
            break
    tr.timers.enabled = not args.no_kernel_timers
    if not tr.graph_active:
        tr.timers.reset()
    launches0 = K.LAUNCHES
    retries0 = torch.cuda.memory_stats(dev).get("num_alloc_retries", 0)
    comp = torch.cuda.current_stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # rank 0 samples its GPU (the line reports rank 0's clocks); one NVML poller
    # per node instead of one per rank keeps driver calls off the other ranks
    # no collector pauses inside the timed loops (the host enqueues the eager
    # multi-rank steps; a GC pause there shows up as an idle GPU)
    gc.collect()
    gc.disable()
    with (sampler if rank == 0 else contextlib.nullcontext(None)) as clocks:
        barrier()
        t0.record(comp)
        marks = [t0]
        for s in range(args.warmup, nsteps):
            tr.step(resident[s])
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(comp)
            marks.append(ev)
        t1.record(comp)
        barrier()
    tr.check_faults()           # a fused-collective barrier timeout voids the run (raises)
    launches = K.LAUNCHES - launches0
    retries_timed = torch.cuda.memory_stats(dev).get("num_alloc_retries", 0) - retries0
    ms = max_over_ranks(t0.elapsed_time(t1)) / args.steps
    # per-step device times (this rank's compute stream), max over ranks per step
    step_ms = torch.tensor([a.elapsed_time(b) for a, b in zip(marks, marks[1:])],
                           device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(step_ms, op=dist.ReduceOp.MAX)
    step_ms = [round(float(x), 2) for x in step_ms]
    kern = {k: tr.timers.summary(k) for k in ("adamw", "accumulate", "gather")}
    kern = {k: v for k, v in kern.items() if v["launches"]}
    steps_timed = 1 if tr.graph_active else args.steps     # graph: the last replay
    tr.timers.enabled = False

    # ---- end to end through the public API with host buffers (e2e) --------
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    loss_val = 0.0
    for s in range(args.warmup, nsteps):
        x = host[s].to(dev, non_blocking=True)
        loss_val = float(tr.step(x))          # D2H read of the step's loss
    e1.record(comp)
    barrier()
    tr.check_faults()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    gc.enable()
    trace_report = None
    if args.trace_dir:
        from paper_2411_01075_b200 import trace as T
        os.makedirs(args.trace_dir, exist_ok=True)
        tr.tracer = T.StepTracer(job.cluster.gpus[rank].id)
        tr.step(resident[-1])
        ev = tr.tracer.collect()
        tr.tracer = None
        T.trace_to_jsonl(ev, os.path.join(args.trace_dir, f"rank{rank}.jsonl"))
        T.trace_to_chrome(ev, os.path.join(args.trace_dir, f"rank{rank}.chrome.json"))
        fwd_l, bwd_l = T.per_layer_metrics(ev, arch.layers)
        trace_report = {"lint_problems": T.lint_measured_trace(ev, arch.layers),
                        "measured_layer_fwd_ms": fwd_l, "measured_layer_bwd_ms": bwd_l,
                        "predicted_layer_fwd_ms": plan.predicted_layer_fwd_ms,
                        "predicted_layer_bwd_ms": plan.predicted_layer_bwd_ms, "events": len(ev)}
        with open(os.path.join(args.trace_dir, f"rank{rank}.report.json"), "w") as fh:
            json.dump(trace_report, fh, indent=1)
    ctx.__exit__(None, None, None)
    # per-rank peak of the caching allocator against the emulated HBM cap
    ms_ = torch.cuda.memory_stats(dev)
    mem = torch.tensor([torch.cuda.max_memory_allocated(dev) / 2 ** 30,
                        emu.memory_cap_bytes / 2 ** 30,
                        torch.cuda.max_memory_reserved(dev) / 2 ** 30,
                        float(ms_.get("num_alloc_retries", 0)), float(retries_timed),
                        float(tr.head_chunk or 0)],
                       device=dev, dtype=torch.float64)
    if world > 1:
        allm = [torch.zeros_like(mem) for _ in range(world)]
        dist.all_gather(allm, mem)
    else:
        allm = [mem]
    # per rank: [peak allocated GiB, cap GiB, peak reserved GiB, allocator retries
    # (whole run), allocator retries inside the device-timed region, head chunk
    # (samples; 0 = whole microbatch)]
    peak_mem = [[round(float(x[0]), 3), round(float(x[1]), 3), round(float(x[2]), 3),
                 int(x[3]), int(x[4]), int(x[5])] for x in allm]
    # every rank's owned-kernel rates (rank 0's are the line's "kernels")
    mine = {k: [v["launches"], round(v["gbs"] or 0.0, 1), round(v["ms_total"] / steps_timed, 4)]
            for k, v in kern.items()}
    if world > 1:
        kern_by_rank = [None] * world
        dist.all_gather_object(kern_by_rank, mine)
    else:
        kern_by_rank = [mine]

    B = plan.total_batch
    hbm, hbm_kind = peaks()
    bf16_peak = bf16_sustained()
    from paper_2411_01075_b200.planner import crosscheck_measured
    xc = crosscheck_measured(plan, ms)
    # dominant owned kernel = the one with the largest share of the timed steps
    if not kern:                              # --no-kernel-timers
        kern = {"adamw": {"launches": 0, "ms_total": 0.0, "ms_mean": 0.0, "bytes_total": 0.0,
                          "bytes_per_launch": 0.0, "gbs": None}}
    dom = max(kern, key=lambda k: kern[k]["ms_total"])
    achieved = kern[dom]["gbs"]
    traffic = traffic_from_profile(dom, kern[dom]["bytes_per_launch"])

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            ref = cpu_reference_rate(args.config, B)
            cpu = {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample")}
        tok_bytes = sum(h.numel() * h.element_size() for h in host[:1]) * world
        line = {
            "metric": "train samples/s", "value": B / (ms * 1e-3), "unit": "samples/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "step_ms": step_ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic tokens (splitmix64), random-init weights",
            "config": {"workload": job.config.name, "description": describe(args.config, world),
                       "global_batch": B, "seq_len": arch.seq,
                       "plan": [[a.microbatch, a.num_microbatches, a.state_ratio]
                                for a in plan.assignments],
                       "uneven_units": plan.unit_shards.uneven_units,
                       "offload_schedule": args.offload_schedule,
                       "peak_vs_cap_gib": peak_mem,
                       # per rank: {kernel: [launches, algorithmic GB/s, ms per step]}
                       "kernels_by_rank": kern_by_rank,
                       "cuda_graph": tr.graph_active,
                       "extra_warmup_steps": extra_warmup,
                       "activation_offload_ranks": [
                           i for i, a in enumerate(plan.assignments)
                           if args.offload == "on" or (args.offload == "auto"
                                                       and a.num_microbatches > 1)],
                       "profiles": ("measured" if any(d.get("profile_key") for d in job.profile_docs)
                                    and not args.analytic_profiles else "analytic"),
                       "planner_predicted_iteration_ms": plan.predicted_iteration_ms,
                       # the reference's crosscheck_optimizer (sim.py:445-452) against the
                       # measured step instead of the simulator
                       "crosscheck": {"predicted_ms": xc.predicted_ms, "measured_ms": xc.measured_ms,
                                      "rel_error": xc.rel_error,
                                      "measured_median_ms": statistics.median(step_ms),
                                      "rel_error_median": abs(statistics.median(step_ms)
                                                              - xc.predicted_ms)
                                      / statistics.median(step_ms)},
                       "parallelism": f"uneven-fsdp{world}",
                       "emulation_rank0": emu.describe(),
                       # sum over ranks of the emulated tiers' SM fractions (N=1: 1.0);
                       # value / tier_capacity is the throughput per full-B200 equivalent
                       "tier_capacity": tier_capacity(job, args.no_emulate),
                       "collectives": route_summary(tr),
                       "symm_ctas": args.symm_ctas,
                       "adamw_overlap": tr.overlap_adamw,
                       "l2": "working set (p,g,m,v,shadow = 30 B/param) >> 126 MB L2; no flush"},
            "e2e": {"value": B / (e2e_ms * 1e-3), "unit": "samples/s",
                    "h2d_bytes_per_step": tok_bytes, "d2h_bytes_per_step": 4 * world},
            "roofline": {"kernel": f"het_{dom}", "bound": "hbm", "achieved": achieved,
                         "peak": hbm, "peak_kind": hbm_kind, "unit": "GB/s",
                         "frac": achieved / hbm if achieved else None, "traffic": traffic,
                         "algorithmic_bytes_per_launch": kern[dom]["bytes_per_launch"],
                         "step_share": kern[dom]["ms_total"] / steps_timed / ms},
            # model FLOPs (6 P T + attention, no recompute) per second against the
            # measured sustained dense bf16 peak: the step-level context of the line
            # (whole job: the peak of all N GPUs; the emulated tiers use fewer SMs, so
            # the per-full-B200-equivalent figure is frac * n_gpus / tier_capacity)
            "mfu": {"model_tflop_per_step": B * arch.model_flops_per_sample() / 1e12,
                    "achieved_tflops": B * arch.model_flops_per_sample() / (ms * 1e-3) / 1e12,
                    "peak_tflops": bf16_peak * world,
                    "frac": B * arch.model_flops_per_sample() / (ms * 1e-3) / 1e12
                    / (bf16_peak * world)},
            "kernels": {k: dict(v, ms_per_step=v["ms_total"] / steps_timed)
                        for k, v in kern.items()},
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
            "loss": loss_val,
        }
        if trace_report is not None:
            line["trace_rank0"] = {k: v for k, v in trace_report.items() if k != "events"}
        print(json.dumps(line), flush=True)
    torch.cuda.synchronize()
    # a captured step holds NCCL graph nodes of comm_ag / comm_rs: destroy it before
    # the communicators (ncclCommDestroy would otherwise wait on the live graph)
    tr.release_graph()
    if world > 1:
        # teardown never costs the run: the line is printed, so a hung NCCL / symmetric
        # memory destructor ends the process after a grace period instead of hanging
        import threading
        threading.Timer(120.0, lambda: os._exit(0)).start()
        dist.barrier()
        comm_ag.close()
        comm_rs.close()
        dist.destroy_process_group()
        sys.stdout.flush()
        sys.stderr.flush()
        os._exit(0)
    if emu.green is not None:
        # The green context must outlive every tensor that touched its stream;
        # interpreter teardown frees them in arbitrary order (and then records
        # events on a destroyed context), so end the process here instead.
        sys.stdout.flush()
        sys.stderr.flush()
        os._exit(0)


if __name__ == "__main__":
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        # tight emulated HBM caps (layered-GA tiers of 1.5-2.5 GiB): expandable
        # segments keep the caching allocator from failing on fragmentation.
        # Set before the first CUDA allocation.
        os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
        try:
            main()
        except BaseException:
            # one failed rank must not leave the others blocked in a collective
            # (or this process in communicator teardown): report and leave at once,
            # so the launcher tears the job down
            import traceback
            traceback.print_exc()
            sys.stderr.flush()
            os._exit(1)
    else:
        main()
