"""Practical NVLink 5 / NVSwitch peak of this box, the denominator the
collective fractions are reported against (beside the 900 GB/s per direction
nominal). Launch with torchrun, one rank per GPU (N >= 2):

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/nvlink_peak.py [--mb 1024]

Measured, 1 GB messages, CUDA events on the issuing stream, median of
--iters after warm-up, max over ranks:
  nccl_allgather      even ncclAllGather (bf16), nccl-tests busbw (n-1)/n S / t
  nccl_reducescatter  even ncclReduceScatter (fp32), same formula
  nccl_allreduce      ncclAllReduce (fp32, through torch), busbw 2 (n-1)/n S / t
  fused_peer_ag       this repo's fused all-gather, peer-store route, even shards
  ce_ring_copy        every rank copies S bytes to its ring successor at once
                      (copy engines, cudaMemcpyPeerAsync through torch): S / t
The practical peak is the largest of them; rank 0 prints one JSON line.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2411_01075_b200 import hetstep as K  # noqa: E402


def timed(fn, iters, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    s = torch.cuda.current_stream()
    ev = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        ev.append((a, b))
    torch.cuda.synchronize()
    ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=float, default=1024)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--ctas", type=int, default=128)
    a = ap.parse_args()
    world, rank, local = (int(os.environ[k]) for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    ids = [K.unique_id()] if rank == 0 else [None]
    dist.broadcast_object_list(ids, src=0)
    comm = K.Comm(ids[0], world, rank)
    S = int(a.mb * (1 << 20))
    out = {}
    try:
        n16 = S // 2 // world * world
        c = [n16 // world] * world
        o = [j * (n16 // world) for j in range(world)]
        send = torch.randn(c[rank], device=dev).to(torch.bfloat16)
        unit = torch.empty(n16, dtype=torch.bfloat16, device=dev)
        ms = timed(lambda: K.allgather_uneven(send, unit, c, o, comm, rank, K.ALGO_EVEN),
                   a.iters, a.warmup)
        out["nccl_allgather"] = (world - 1) / world * (2 * n16) / (ms * 1e-3) / 1e9
        n32 = S // 4 // world * world
        c32 = [n32 // world] * world
        o32 = [j * (n32 // world) for j in range(world)]
        src = torch.randn(n32, device=dev)
        shard = torch.empty(c32[rank], device=dev)
        ms = timed(lambda: K.reduce_scatter_uneven(src, shard, c32, o32, comm, rank,
                                                   K.ALGO_EVEN), a.iters, a.warmup)
        out["nccl_reducescatter"] = (world - 1) / world * (4 * n32) / (ms * 1e-3) / 1e9
        ms = timed(lambda: dist.all_reduce(src), a.iters, a.warmup)
        out["nccl_allreduce"] = 2 * (world - 1) / world * (4 * n32) / (ms * 1e-3) / 1e9
        del src, shard
        ws = K.SymmWorkspace([("unit", n16, torch.bfloat16)], dist.group.WORLD.group_name, dev,
                             rank, world, ctas=a.ctas, use_multicast=False, policy=K.SYMM_PEER)
        mine = torch.randn(c[rank], device=dev)
        ms = timed(lambda: ws.allgather_pack(mine, "unit", 0, c, o), a.iters, a.warmup)
        out["fused_peer_ag"] = (world - 1) / world * (2 * n16) / (ms * 1e-3) / 1e9
        del ws
        # copy-engine ring: every rank writes S bytes into its successor's buffer
        buf = torch.empty(S, dtype=torch.uint8, device=dev)
        dst = [torch.empty(S, dtype=torch.uint8, device=torch.device("cuda", j))
               if j == (local + 1) % world else None for j in range(world)]
        peer = dst[(local + 1) % world]
        if peer is not None:
            try:
                ms = timed(lambda: peer.copy_(buf, non_blocking=True), a.iters, a.warmup)
                out["ce_ring_copy"] = S / (ms * 1e-3) / 1e9
            except RuntimeError:
                pass
        status = K.SymmWorkspace.status()
        if rank == 0:
            best = max(out.values())
            print(json.dumps({"n_gpus": world, "message_mb": a.mb, "measured_gbs": out,
                              "practical_peak_gbs": best,
                              "practical_peak_from": max(out, key=out.get),
                              "nominal_gbs": 900.0, "symm_status": status,
                              "method": "CUDA events, median of %d after %d warm-up, max over "
                                        "ranks (tools/nvlink_peak.py)" % (a.iters, a.warmup)}),
                  flush=True)
    finally:
        comm.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
