"""Worker for the world_size-2 gloo tests of the step driver (CPU, fake
kernels). Runs one rank: builds its RankLayout from the shared plan, runs one
Cephalo step, and returns the all-gathered full fp32 units it ends with."""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def run_rank(rank: int, world: int, port: int, plan_doc: dict, arch_name: str, units, steps,
             out_q) -> None:
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _body(rank, world, plan_doc, arch_name, units, steps, out_q)
    except BaseException:            # surface worker failures instead of a queue timeout
        import traceback
        out_q.put((rank, {"error": traceback.format_exc()}))
        raise
    finally:
        dist.destroy_process_group()


def _body(rank, world, plan_doc, arch_name, units, steps, out_q):
    import torch
    import torch.distributed as dist

    import fake_kernels
    from paper_2411_01075_b200 import plan_from_dict
    from paper_2411_01075_b200 import step as S
    from paper_2411_01075_b200.data import rank_tokens
    from paper_2411_01075_b200.model import ARCHS
    S.K = fake_kernels
    arch = ARCHS[arch_name]
    plan = plan_from_dict(plan_doc)
    comm = fake_kernels.Comm(b"", world, rank)
    tr = S.UnevenFSDPTrainer(arch, plan, rank, comm_ag=comm, comm_rs=comm,
                             device=torch.device("cpu"))
    tr.load_full_units(units)
    losses = []
    for s in range(steps):
        tok = rank_tokens(plan, rank, arch.seq, arch.vocab, seed=11, step=s)
        losses.append(tr.step(torch.from_numpy(tok)))
    loss = torch.stack(losses) if losses else torch.zeros(0)
    dist.all_reduce(loss)
    # numpy copies: tensors in a Queue would be shared by fd and die with the worker
    g = [t.numpy().copy() for t in tr.full_units("g32")]
    p = [t.numpy().copy() for t in tr.full_units("p32")]
    out_q.put((rank, {"g": g, "p": p, "loss": loss.tolist(),
                      "owned": tr.L.owned_params, "calls": list(fake_kernels.calls)}))
