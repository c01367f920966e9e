#!/usr/bin/env python
"""Uneven all-gather / reduce-scatter sweep (BASELINE.json config 5: "uneven
all-gather/reduce-scatter + AdamW sweep, 1 MB-1 GB shard skews at 2/4/8
GPUs"). Launch with torchrun, one rank per GPU:

  torchrun --nproc-per-node N --master-addr 127.0.0.1 bench_collectives.py [--sizes-mb ...]

For a unit of S bytes split into per-rank ranges s_i, the reported bus
bandwidth is max_i(S - s_i) / t — the bytes the most-loaded rank must ingest
(SURVEY.md §8d); for an even split it equals nccl-tests' (n-1)/n * S / t,
which is reported beside it. Times are CUDA events on the issuing stream,
median of `--iters` after warm-up, max over ranks. Rank 0 prints one JSON
line per (op, size, skew, algo) and a final summary line.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2411_01075_b200 import hetstep as K  # noqa: E402
from paper_2411_01075_b200.configs import build_job  # noqa: E402

ALGOS = {"auto": K.ALGO_AUTO, "p2p": K.ALGO_P2P, "owner": K.ALGO_OWNER,
         "symm": "symm", "symm_mc": "symm_mc", "symm_peer": "symm_peer", "route": "route",
         "symm_relay": "symm_relay", "symm_helpers": "symm_helpers",
         "symm_helpers_mc": "symm_helpers_mc",
         "symm_bf16wire": "symm_bf16wire", "symm_bf16wire_helpers": "symm_bf16wire_helpers"}
SYMM = {"symm": (True, K.SYMM_AUTO), "symm_mc": (True, K.SYMM_MULTICAST),
        "symm_peer": (False, K.SYMM_PEER), "symm_relay": (False, K.SYMM_RELAY),
        "symm_helpers": (False, K.SYMM_HELPERS), "symm_helpers_mc": (True, K.SYMM_HELPERS_MC)}


def skew_counts(skew: str, total: int, n: int) -> list[int]:
    if skew == "even":
        base = [total // n] * n
        base[-1] += total - sum(base)
        return base
    if skew == "single_owner":
        return [total] + [0] * (n - 1)
    if skew == "two_to_one":      # alternating 2:1 weights
        w = [2 if i % 2 == 0 else 1 for i in range(n)]
    elif skew == "geometric":     # 1, 1/2, 1/4, ...
        w = [2.0 ** -i for i in range(n)]
    else:
        raise ValueError(skew)
    c = [int(total * x / sum(w)) for x in w]
    c[0] += total - sum(c)
    return c


def offsets(c):
    out, pos = [], 0
    for x in c:
        out.append(pos)
        pos += x
    return out


def time_op(fn, iters: int, warmup: int) -> float:
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    ts = []
    s = torch.cuda.current_stream()
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        ts.append((a, b))
    torch.cuda.synchronize()
    ms = float(np.median([a.elapsed_time(b) for a, b in ts]))
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-mb", type=float, nargs="*", default=[1, 4, 16, 64, 256, 1024])
    ap.add_argument("--skews", nargs="*",
                    default=["even", "two_to_one", "geometric", "single_owner", "planner"])
    ap.add_argument("--algos", nargs="*", default=["route", "auto", "owner", "p2p", "symm",
                                                   "symm_mc", "symm_peer"])
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--planner-config", default="llama_1b3")
    ap.add_argument("--ctas", type=int, default=128)
    args = ap.parse_args()

    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), \
        int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    ids = [K.unique_id()] if rank == 0 else [None]
    dist.broadcast_object_list(ids, src=0)
    comm = K.Comm(ids[0], world, rank)
    job = build_job(args.planner_config, world)
    planner_ratio = [a.state_ratio for a in job.plan.assignments]
    best: dict[str, float] = {}
    maxel = int(max(args.sizes_mb) * (1 << 20)) // 2 + 64
    ws = {}
    for an, (mc, policy) in SYMM.items():
        if an in args.algos or (an == "symm_helpers" and "symm_bf16wire_helpers" in args.algos) \
                or (an in ("symm", "symm_relay", "symm_helpers", "symm_helpers_mc")
                    and world > 2 and
                                "route" in args.algos) or (an == "symm" and (
                                    "route" in args.algos or "symm_bf16wire" in args.algos)):
            ws[an] = K.SymmWorkspace([("unit", maxel, torch.bfloat16), ("acc", maxel + 64,
                                                                         torch.float32),
                                      ("g16", maxel + 64, torch.bfloat16)],
                                     dist.group.WORLD.group_name, dev, rank, world,
                                     ctas=args.ctas, use_multicast=mc, policy=policy)
            if rank == 0:
                print(json.dumps({"workspace": an, "multicast": ws[an].multicast}), flush=True)
    try:
        for op in ("allgather", "reduce_scatter"):
            esize = 2 if op == "allgather" else 4
            for mb in args.sizes_mb:
                total = int(mb * (1 << 20)) // esize
                for skew in args.skews:
                    if skew == "planner":
                        c = [int(total * r) for r in planner_ratio]
                        c[int(np.argmax(c))] += total - sum(c)
                    else:
                        c = skew_counts(skew, total, world)
                    o = offsets(c)
                    for an in args.algos:
                        algo = ALGOS[an]
                        if op == "reduce_scatter" and algo in (K.ALGO_P2P, "symm_relay"):
                            continue
                        if op == "allgather" and algo == "symm_helpers_mc":   # fp32 RS only
                            continue
                        if algo == "route":   # the train step's per-unit choice
                            pick = K.route_collective("ag" if op == "allgather" else "rs", c,
                                                      world, "symm" in ws)
                            algo = "symm" if pick == "symm" else K.ALGO_AUTO
                            if algo == "symm":
                                pol = K.symm_policy("ag" if op == "allgather" else "rs", c,
                                                    world, multicast=ws["symm"].multicast)
                                algo = {K.SYMM_RELAY: "symm_relay",
                                        K.SYMM_HELPERS: "symm_helpers",
                                        K.SYMM_HELPERS_MC: "symm_helpers_mc"}.get(pol, "symm")
                        if algo in ("symm_bf16wire", "symm_bf16wire_helpers"):
                            if op != "reduce_scatter":
                                continue
                            hel = algo == "symm_bf16wire_helpers"
                            w = ws["symm_helpers" if hel else "symm"]
                            w["g16"][:total].normal_()
                            out = torch.empty(c[rank], device=dev)
                            wts = [1.0 / world] * world
                            pol = K.SYMM_HELPERS if hel else K.SYMM_AUTO
                            st_ = "acc" if hel else None
                            fn = lambda: w.reduce_scatter_bf16("g16", 0, out, c, o, wts,  # noqa: E731
                                                               policy=pol, stage=st_)
                        elif isinstance(algo, str):
                            w = ws[algo]
                            if op == "allgather":
                                src32 = torch.randn(c[rank], device=dev)
                                fn = lambda: w.allgather_pack(src32, "unit", 0, c, o)  # noqa: E731
                            else:
                                w["acc"][:total].normal_()
                                out = torch.empty(c[rank], device=dev)
                                fn = lambda: w.reduce_scatter("acc", 0, out, c, o)  # noqa: E731
                        elif op == "allgather":
                            send = torch.randn(c[rank], device=dev).to(torch.bfloat16)
                            unit = torch.empty(total, dtype=torch.bfloat16, device=dev)
                            fn = lambda: K.allgather_uneven(send, unit, c, o, comm, rank, algo)  # noqa: E731
                        else:
                            src = torch.randn(total, device=dev)
                            out = torch.empty(c[rank], device=dev)
                            fn = lambda: K.reduce_scatter_uneven(src, out, c, o, comm, rank, algo)  # noqa: E731
                        ms = time_op(fn, args.iters, args.warmup)
                        # bus bytes of the fp32 result (the bf16 wire moves half of them)
                        S = total * esize
                        ingest = max(S - x * esize for x in c)
                        bus = ingest / (ms * 1e-3) / 1e9
                        nccl_bus = (world - 1) / world * S / (ms * 1e-3) / 1e9
                        key = f"{op}/{skew}"
                        if mb >= 256 and bus > best.get(key, (0.0, ""))[0]:
                            best[key] = (bus, an)
                        if rank == 0:
                            print(json.dumps({"op": op, "n_gpus": world, "size_mb": mb,
                                              "skew": skew, "algo": an, "ms": ms,
                                              "bus_gbs": bus, "nccl_tests_bus_gbs": nccl_bus,
                                              "counts": c if world <= 8 else None}), flush=True)
                        del fn
        status = K.SymmWorkspace.status() if ws else 0
        if rank == 0:
            print(json.dumps({"summary": "best bus GB/s at >= 256 MB", "n_gpus": world,
                              "symm_status": status,
                              "best": best,
                              "frac_of_770": {k: v[0] / 770.0 for k, v in best.items()}}),
                  flush=True)
    finally:
        comm.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
