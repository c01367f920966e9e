"""torchrun worker of tests/test_multigpu_configs.py: one train step of the
bench plan of each BASELINE config at this world size, on real GPUs through
the fused collectives, with every microbatch scaled down so the fp32 CPU
oracle finishes in seconds (the plan's state layout, l_i and Eq. 1 weights are
kept). Rank 0 writes OUT_DIR/<config>.npz: the reduced full-unit gradients,
the post-step masters, the tokens and the plan.

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/mgpu_config_worker.py OUT_DIR
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2411_01075_b200 import GpuAssignment, TrainPlan, assign_unit_shards  # noqa: E402
from paper_2411_01075_b200 import hetstep as K  # noqa: E402
from paper_2411_01075_b200.configs import build_job  # noqa: E402
from paper_2411_01075_b200.data import rank_tokens  # noqa: E402
from paper_2411_01075_b200.model import init_flat  # noqa: E402
from paper_2411_01075_b200.step import UnevenFSDPTrainer  # noqa: E402

CASES = {2: ["gpt2_small", "llama_1b3"], 4: ["gpt2_small", "bert_large", "llama_1b3"],
         8: ["gpt2_small", "bert_large", "llama_1b3"]}
TARGET = {"gpt2_small": 8, "bert_large": 8, "llama_1b3": 4}


def scaled_plan(name: str, n: int):
    """The bench plan at n ranks with microbatches scaled so B ~ TARGET[name]."""
    job = build_job(name, n, measured=True)
    k = max(1, math.ceil(job.plan.total_batch / TARGET[name]))
    ratios = [a.state_ratio for a in job.plan.assignments]
    asg = []
    for a in job.plan.assignments:
        m = 0 if a.microbatch == 0 else max(1, a.microbatch // k)
        asg.append((m, a.num_microbatches if m else 0))
    arch = job.arch
    model = arch.model_spec(sum(m * l for m, l in asg))
    plan = TrainPlan(tuple(GpuAssignment(f"g{i}", m, l, m * l, r, 0.0, r * model.state_bytes)
                           for i, ((m, l), r) in enumerate(zip(asg, ratios))),
                     1.0, 1.0, 2.0 * arch.layers, True, assign_unit_shards(ratios, model))
    assert [list(r) for r in plan.unit_shards.shards] == \
        [list(r) for r in job.plan.unit_shards.shards]      # the bench layout itself
    return arch, plan


def cpu_units(arch, seed):
    units = []
    for u in range(arch.layers + 1):
        g = torch.Generator().manual_seed(seed * 100003 + u)
        units.append(init_flat(arch.root_layout() if u == arch.layers else arch.unit_layout(),
                               g, "cpu"))
    return units


def main(out_dir: str) -> None:
    world, rank, local = (int(os.environ[k]) for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    ids = [K.unique_id(), K.unique_id()] if rank == 0 else [None, None]
    dist.broadcast_object_list(ids, src=0)
    cag, crs = K.Comm(ids[0], world, rank), K.Comm(ids[1], world, rank)
    try:
        # each config twice: the route table the bench uses ("default": every unit
        # on the fused kernels) and the NCCL ring for near-single-owner units at
        # N >= 4 ("nccl": hetstep.OWNER_FUSED = "none")
        for name, mode in [(c, m) for c in CASES.get(world, []) for m in ("default", "nccl")]:
            K.OWNER_FUSED = "none" if mode == "nccl" else "all"
            arch, plan = scaled_plan(name, world)
            units = cpu_units(arch, seed=3)
            tr = UnevenFSDPTrainer(arch, plan, rank, comm_ag=cag, comm_rs=crs, device=dev,
                                   algo=K.ALGO_SYMM)
            tr.load_full_units(units)
            p0 = [t.cpu().numpy() for t in tr.full_units("p32")]
            toks = [rank_tokens(plan, r, arch.seq, arch.vocab, seed=21, step=0)
                    for r in range(world)]
            loss = tr.step(torch.from_numpy(toks[rank]).to(dev))
            tr.check_faults()
            dist.all_reduce(loss)
            g = [t.cpu().numpy() for t in tr.full_units("g32")]
            p = [t.cpu().numpy() for t in tr.full_units("p32")]
            info = dict(route_ok=float(tr.route_check["ok"]),
                        fused=float(all(r == "symm" for r in tr.ag_route + tr.rs_route)),
                        helpers=float(sum(1 for x in tr.ag_policy + tr.rs_policy
                                          if x == K.SYMM_HELPERS)),
                        wire16=float(sum(tr.wire16)), status=float(K.SymmWorkspace.status()))
            if rank == 0:
                np.savez(os.path.join(out_dir, f"{name}.{mode}.npz"), loss=float(loss),
                         micro=np.array([(a.microbatch, a.num_microbatches)
                                         for a in plan.assignments]),
                         ratios=np.array([a.state_ratio for a in plan.assignments]),
                         toks=np.stack([np.pad(t, ((0, max(len(x) for x in toks) - len(t)),
                                                   (0, 0))) for t in toks]),
                         tok_rows=np.array([len(t) for t in toks]),
                         **{f"g{u}": x for u, x in enumerate(g)},
                         **{f"p{u}": x for u, x in enumerate(p)},
                         **{f"p0_{u}": x for u, x in enumerate(p0)}, **info)
            del tr
            torch.cuda.empty_cache()
            dist.barrier()
    finally:
        K.OWNER_FUSED = "all"
        cag.close()
        crs.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
