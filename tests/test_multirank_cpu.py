"""N>1 host logic over gloo on CPU (world_size 2): each rank builds its own
RankLayout from the shared plan, all-gathers its units, runs its l_i
microbatches, reduce-scatters Eq. 1-weighted gradients into its uneven
shard and applies AdamW to it. Kernels are the oracle-backed test double;
the assembled result must equal the single-process oracle step."""
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import mr_worker
from oracle import model_oracle as MO
from oracle import step_oracle as SO
from oracle.tolerances import BF16_GRAD_RTOL, FP32_RTOL, max_rel, norm_rel
from paper_2411_01075_b200 import (GpuAssignment, ModelSpec, TrainPlan, assign_unit_shards,
                                   plan_to_dict)
from paper_2411_01075_b200.configs import build_job
from paper_2411_01075_b200.data import rank_tokens
from paper_2411_01075_b200.model import ARCHS, init_flat


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _units(arch):
    out = []
    for u in range(arch.layers + 1):
        g = torch.Generator().manual_seed(17 + u)
        out.append(init_flat(arch.root_layout() if u == arch.layers else arch.unit_layout(), g,
                             "cpu"))
    return out


def _plan(arch, micro, ratios):
    B = sum(m * l for m, l in micro)
    model = ModelSpec(arch.layers, arch.unit_params, B)
    rows = tuple(GpuAssignment(f"g{i}", m, l, m * l, r, 0.0, r * model.state_bytes)
                 for i, ((m, l), r) in enumerate(zip(micro, ratios)))
    return TrainPlan(rows, 1.0, 1.0, 2.0 * arch.layers, True, assign_unit_shards(ratios, model))


def _run(plan, arch, units, steps=1, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=mr_worker.run_rank,
                         args=(r, world, port, plan_to_dict(plan), arch.name, units, steps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for r, d in res.items():
        assert "error" not in d, f"rank {r} failed:\n{d['error']}"
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


PLANS = {
    "mixed": ([(2, 2), (1, 3)], [683 / 1024, 341 / 1024]),      # l_i > 1 on both, mixed shards
    "single_owner": ([(3, 1), (1, 2)], [1.0, 0.0]),             # every unit owned by rank 0
    "idle_rank": ([(4, 1), (0, 0)], [0.5, 0.5]),                # rank 1 computes nothing
}


@pytest.mark.parametrize("case", sorted(PLANS))
def test_two_rank_step_equals_oracle(case):
    arch = ARCHS["tiny_gpt"]
    micro, ratios = PLANS[case]
    plan = _plan(arch, micro, ratios)
    units = _units(arch)
    res = _run(plan, arch, units)
    r0, r1 = res[0], res[1]
    # both ranks assemble identical full vectors
    for a, b in zip(r0["g"] + r0["p"], r1["g"] + r1["p"]):
        assert np.array_equal(a, b)
    assert r0["owned"] + r1["owned"] == arch.layers * arch.unit_params + arch.root_params
    toks = [rank_tokens(plan, i, arch.seq, arch.vocab, seed=11, step=0) for i in range(2)]
    live = [(t, mi) for t, mi in zip(toks, micro) if mi[0] > 0]
    gu, gr, loss = MO.weighted_gradient(arch, units[:-1], units[-1], [t for t, _ in live],
                                        [mi for _, mi in live])
    assert abs(r0["loss"][0] - loss) <= BF16_GRAD_RTOL * abs(loss)
    for u, ref in enumerate(gu + [gr]):
        assert norm_rel(r0["g"][u], ref.numpy()) <= BF16_GRAD_RTOL, f"unit {u}"
    opt = dict(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1)
    for u, full in enumerate(units):
        z = np.zeros(full.numel(), np.float32)
        rp, _, _ = SO.adamw(full.numpy(), r0["g"][u], z, z, step=1, **opt)
        assert max_rel(r0["p"][u], rp) <= FP32_RTOL
    if case == "idle_rank":
        assert "accumulate" not in r1["calls"]
    assert r1["calls"].count("reduce_scatter") == arch.layers + 1


def test_planner_job_two_ranks_two_steps():
    """The planner's own 2-rank plan (single-owner units) over two steps: the
    second step all-gathers the AdamW-updated bf16 shadow."""
    job = build_job("tiny_gpt", 2, global_batch=6)
    arch, plan = job.arch, job.plan
    units = _units(arch)
    res = _run(plan, arch, units, steps=2)
    cpu = MO.CPUStep(arch, units[:-1], units[-1],
                     dict(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1))
    micro = [(a.microbatch, a.num_microbatches) for a in plan.assignments]
    for s in range(2):
        toks = [rank_tokens(plan, i, arch.seq, arch.vocab, seed=11, step=s) for i in range(2)]
        ref = cpu.step(toks, micro)
        assert abs(res[0]["loss"][s] - ref) <= BF16_GRAD_RTOL * abs(ref)


def test_planner_job_eight_ranks():
    """The 8-rank plan the bench's N=8 run uses (4 state owners, 4 zero-shard
    ranks, 2:1 micro-batches): the host logic of the widest world size, which
    the GPU pool here cannot host, against the oracle."""
    job = build_job("tiny_gpt", 8)
    arch, plan = job.arch, job.plan
    assert len(plan.assignments) == 8
    units = _units(arch)
    res = _run(plan, arch, units, steps=1, world=8)
    for r in range(1, 8):
        for a, b in zip(res[0]["g"] + res[0]["p"], res[r]["g"] + res[r]["p"]):
            assert np.array_equal(a, b)
    assert sum(res[r]["owned"] for r in range(8)) == \
        arch.layers * arch.unit_params + arch.root_params
    micro = [(a.microbatch, a.num_microbatches) for a in plan.assignments]
    toks = [rank_tokens(plan, i, arch.seq, arch.vocab, seed=11, step=0) for i in range(8)]
    gu, gr, loss = MO.weighted_gradient(arch, units[:-1], units[-1], toks, micro)
    assert abs(res[0]["loss"][0] - loss) <= BF16_GRAD_RTOL * abs(loss)
    for u, ref in enumerate(gu + [gr]):
        assert norm_rel(res[0]["g"][u], ref.numpy()) <= BF16_GRAD_RTOL, f"unit {u}"
