"""torchrun worker for the multi-GPU parity tests (real kernels + NCCL).

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/mgpu_worker.py OUT_DIR

Rank r checks the uneven all-gather (bit-exact, every algorithm) and the
uneven reduce-scatter (fp32, vs the oracle sum) on a set of shard shapes —
even, ragged-even, single-owner, mixed, zero-count ranks — then runs one
train step of tiny GPT under a mixed uneven plan and writes its results to
OUT_DIR/rank{r}.npz for the parent test to compare with the CPU oracle.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import step_oracle as O  # noqa: E402
from oracle.tolerances import max_rel  # noqa: E402
from paper_2411_01075_b200 import (GpuAssignment, ModelSpec, TrainPlan,  # noqa: E402
                                   assign_unit_shards)
from paper_2411_01075_b200 import hetstep as K  # noqa: E402
from paper_2411_01075_b200.data import rank_tokens  # noqa: E402
from paper_2411_01075_b200.model import ARCHS, init_flat  # noqa: E402
from paper_2411_01075_b200.step import UnevenFSDPTrainer  # noqa: E402


def shard_cases(n: int) -> list[list[int]]:
    cases = [[1000] * n, [1001] * (n - 1) + [999], [4096 * 7 + 3] + [0] * (n - 1),
             [0] * (n - 1) + [12345], [3_571_623] + [3_516_249] * (n - 1)]
    rng = np.random.default_rng(n)
    cases.append([int(x) for x in rng.integers(0, 50_000, size=n)])
    return [c for c in cases if sum(c) > 0]


def offsets(c):
    return [int(sum(c[:j])) for j in range(len(c))]


def stage(rank: int, what: str) -> None:
    print(f"[rank {rank}] {what}", file=sys.stderr, flush=True)


def main(out_dir: str) -> None:
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    import faulthandler
    # a hung rank dumps every thread's Python stack (then keeps running)
    faulthandler.dump_traceback_later(int(os.environ.get("HET_WORKER_DUMP_S", "240")),
                                      repeat=True, file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    ids = [K.unique_id(), K.unique_id()] if rank == 0 else [None, None]
    dist.broadcast_object_list(ids, src=0)
    cag, crs = K.Comm(ids[0], world, rank), K.Comm(ids[1], world, rank)
    report = {}
    try:
        stage(rank, "nccl collectives")
        for ci, counts in enumerate(shard_cases(world)):
            offs = offsets(counts)
            total = sum(counts)
            full = np.random.default_rng(ci).standard_normal(total).astype(np.float32)
            bits = O.pack(full)
            mine = torch.from_numpy(full[offs[rank]:offs[rank] + counts[rank]]).to(dev)
            send = torch.empty(counts[rank], dtype=torch.bfloat16, device=dev)
            K.pack_bf16(mine, send)
            for algo in (K.ALGO_AUTO, K.ALGO_P2P, K.ALGO_OWNER):
                unit = torch.empty(total, dtype=torch.bfloat16, device=dev)
                K.allgather_uneven(send, unit, counts, offs, cag, rank, algo)
                torch.cuda.synchronize()
                got = unit.view(torch.int16).cpu().numpy().view(np.uint16)
                report[f"ag{ci}_{algo}"] = int(np.array_equal(got, bits))
            srcs = [np.random.default_rng(100 * ci + r).standard_normal(total).astype(np.float32)
                    for r in range(world)]
            want = O.reduce_scatter(srcs, counts, offs)[rank]
            for algo in (K.ALGO_AUTO, K.ALGO_OWNER):
                out = torch.empty(counts[rank], dtype=torch.float32, device=dev)
                K.reduce_scatter_uneven(torch.from_numpy(srcs[rank]).to(dev), out, counts, offs,
                                        crs, rank, algo)
                torch.cuda.synchronize()
                err = max_rel(out.cpu().numpy(), want) if counts[rank] else 0.0
                report[f"rs{ci}_{algo}"] = float(err)

        stage(rank, "fused collectives")
        # fused symmetric-memory collectives (NVLS multicast when available, then peer)
        maxu = max(sum(c) for c in shard_cases(world)) + 64
        for use_mc, policy in ((True, K.SYMM_MULTICAST), (True, K.SYMM_AUTO), (False, K.SYMM_AUTO),
                               (False, K.SYMM_RELAY), (False, K.SYMM_HELPERS),
                               (True, K.SYMM_HELPERS_MC)):
            ws = K.SymmWorkspace([("unit", maxu, torch.bfloat16), ("acc", maxu, torch.float32),
                                  ("g16", maxu, torch.bfloat16)],
                                 dist.group.WORLD.group_name, dev, rank, world,
                                 use_multicast=use_mc, policy=policy)
            use_mc = f"{int(use_mc)}{policy}"
            report[f"symm_mc_available_{use_mc}"] = float(ws.multicast)
            stage(rank, f"workspace {use_mc} multicast={ws.multicast}")
            for ci, counts in enumerate(shard_cases(world)):
                offs = offsets(counts)
                total = sum(counts)
                full = np.random.default_rng(ci).standard_normal(total).astype(np.float32)
                mine = torch.from_numpy(full[offs[rank]:offs[rank] + counts[rank]]).to(dev)
                for shift in (0, 3):        # unit placed at an odd element offset too
                    ws["unit"].zero_()
                    ws.allgather_pack(mine, "unit", 8 * shift, counts, offs)
                    torch.cuda.synchronize()
                    got = ws["unit"][8 * shift:8 * shift + total].view(torch.int16).cpu().numpy()
                    report[f"symm_ag{ci}_{use_mc}_{shift}"] = int(
                        np.array_equal(got.view(np.uint16), O.pack(full)))
                srcs = [np.random.default_rng(100 * ci + r).standard_normal(total).astype(np.float32)
                        for r in range(world)]
                want = O.reduce_scatter(srcs, counts, offs)[rank]
                ws["acc"][:total].copy_(torch.from_numpy(srcs[rank]))
                out = torch.empty(counts[rank], dtype=torch.float32, device=dev)
                ws.reduce_scatter("acc", 0, out, counts, offs, end_barrier=True)
                torch.cuda.synchronize()
                report[f"symm_rs{ci}_{use_mc}"] = float(
                    max_rel(out.cpu().numpy(), want) if counts[rank] else 0.0)
                # bf16 wire: unscaled bf16 gradients, Eq. 1 weights applied in the RS;
                # expected = sum_j fl32(w_j * g_j) in rank order (IEEE fp32 in numpy)
                wts = [0.0 if r == 1 and world > 2 else (r + 1) / (world * (world + 1) / 2)
                       for r in range(world)]
                g16 = [torch.from_numpy(x).to(torch.bfloat16) for x in srcs]
                ws["g16"][:total].copy_(g16[rank].to(dev))
                want16 = np.zeros(total, np.float32)
                for r in range(world):
                    if wts[r] != 0.0:
                        want16 = want16 + np.float32(wts[r]) * g16[r].float().numpy()
                lo = offs[rank]
                out16 = torch.empty(counts[rank], dtype=torch.float32, device=dev)
                torch.cuda.synchronize()
                dist.barrier()
                ws.reduce_scatter_bf16("g16", 0, out16, counts, offs, wts, end_barrier=True,
                                       policy=policy if policy == K.SYMM_HELPERS else K.SYMM_AUTO,
                                       stage="acc" if policy == K.SYMM_HELPERS else None)
                torch.cuda.synchronize()
                report[f"bf16wire_rs{ci}_{use_mc}"] = int(np.array_equal(
                    out16.cpu().numpy(), want16[lo:lo + counts[rank]]))
            report[f"symm_status_{use_mc}"] = float(K.SymmWorkspace.status(reset=True))
            dist.barrier()
            del ws

        stage(rank, "nccl-route step")
        # one train step under a mixed uneven plan with l_i > 1 on some ranks
        arch = ARCHS["tiny_gpt"]
        micro = [(2, 2), (1, 3), (3, 1), (0, 0), (2, 1), (1, 1), (4, 1), (1, 2)][:world]
        if world == 2:
            micro = [(2, 2), (1, 3)]
        raw = [683, 341, 0, 512, 100, 7, 300, 81][:world]
        ratios = [r / sum(raw) for r in raw]
        ratios[-1] = 1.0 - sum(ratios[:-1])
        B = sum(m * l for m, l in micro)
        model = ModelSpec(arch.layers, arch.unit_params, B)
        plan = TrainPlan(tuple(GpuAssignment(f"g{i}", m, l, m * l, r, 0.0, r * model.state_bytes)
                               for i, ((m, l), r) in enumerate(zip(micro, ratios))),
                         1.0, 1.0, 2.0 * arch.layers, True, assign_unit_shards(ratios, model))
        units = []
        for u in range(arch.layers + 1):
            g = torch.Generator().manual_seed(17 + u)
            units.append(init_flat(arch.root_layout() if u == arch.layers else
                                   arch.unit_layout(), g, "cpu"))
        tr = UnevenFSDPTrainer(arch, plan, rank, comm_ag=cag, comm_rs=crs, device=dev)
        tr.load_full_units(units)
        tok = rank_tokens(plan, rank, arch.seq, arch.vocab, seed=11, step=0)
        loss = tr.step(torch.from_numpy(tok).to(dev))
        dist.all_reduce(loss)
        g = [t.cpu().numpy() for t in tr.full_units("g32")]
        p = [t.cpu().numpy() for t in tr.full_units("p32")]
        stage(rank, "fused-route step")
        # the same step through the fused symmetric-memory (NVLS) collectives
        trs = UnevenFSDPTrainer(arch, plan, rank, comm_ag=cag, comm_rs=crs, device=dev,
                                algo=K.ALGO_SYMM)
        report["symm_route_check_ok"] = float(trs.route_check["ok"] and
                                              trs.route_check["checked"] > 0)
        trs.load_full_units(units)
        from paper_2411_01075_b200.trace import StepTracer, lint_measured_trace
        trs.tracer = StepTracer(f"g{rank}")
        loss_s = trs.step(torch.from_numpy(tok).to(dev))
        report["trace_lint_problems"] = float(len(lint_measured_trace(trs.tracer.collect(),
                                                                      arch.layers)))
        trs.tracer = None
        dist.all_reduce(loss_s)
        gs = [t.cpu().numpy() for t in trs.full_units("g32")]
        ps = [t.cpu().numpy() for t in trs.full_units("p32")]
        report["symm_status_step"] = float(K.SymmWorkspace.status(reset=True))
        stage(rank, "bf16-wire pair steps")
        # l_i <= 1 on every rank: the bf16-wire reduce-scatter against the fp32 one
        pmicro = [(3, 1), (2, 1), (1, 1), (0, 0)][:world] if world > 2 else [(3, 1), (2, 1)]
        pB = sum(m * l for m, l in pmicro)
        pmodel = ModelSpec(arch.layers, arch.unit_params, pB)
        pplan = TrainPlan(tuple(GpuAssignment(f"g{i}", m, l, m * l, r, 0.0, r * pmodel.state_bytes)
                                for i, ((m, l), r) in enumerate(zip(pmicro, ratios))),
                          1.0, 1.0, 2.0 * arch.layers, True, assign_unit_shards(ratios, pmodel))
        ptok = torch.from_numpy(rank_tokens(pplan, rank, arch.seq, arch.vocab, seed=13,
                                            step=0)).to(dev)
        pair = {}
        for wire in (True, False):
            t2 = UnevenFSDPTrainer(arch, pplan, rank, comm_ag=cag, comm_rs=crs, device=dev,
                                   algo=K.ALGO_SYMM, bf16_wire=wire)
            t2.load_full_units(units)
            if wire:
                report["bf16_wire_units"] = float(sum(t2.wire16))
            t2.step(ptok)
            pair[wire] = [t.cpu().numpy() for t in t2.full_units("g32")]
            del t2
        report["symm_status_pair"] = float(K.SymmWorkspace.status(reset=True))

        # odd block count in pair mode: a 3-block model's last group is
        # unit 0 alone, whose accumulate must wait for RS(1)'s end barrier too
        from paper_2411_01075_b200.model import ArchSpec
        arch3 = ArchSpec("tiny_gpt3", "gpt", d=256, layers=3, heads=4, ffn=1024, vocab=4096,
                         seq=128)
        m3 = ModelSpec(arch3.layers, arch3.unit_params, pB)
        plan3 = TrainPlan(tuple(GpuAssignment(f"g{i}", m, l, m * l, r, 0.0, r * m3.state_bytes)
                                for i, ((m, l), r) in enumerate(zip(pmicro, ratios))),
                          1.0, 1.0, 2.0 * arch3.layers, True, assign_unit_shards(ratios, m3))
        units3 = []
        for u in range(arch3.layers + 1):
            g3 = torch.Generator().manual_seed(71 + u)
            units3.append(init_flat(arch3.root_layout() if u == arch3.layers else
                                    arch3.unit_layout(), g3, "cpu"))
        tok3 = rank_tokens(plan3, rank, arch3.seq, arch3.vocab, seed=17, step=0)
        t3 = UnevenFSDPTrainer(arch3, plan3, rank, comm_ag=cag, comm_rs=crs, device=dev,
                               algo=K.ALGO_SYMM)
        report["odd_pair_mode"] = float(t3.pair_units and t3.L.blocks % 2 == 1)
        t3.load_full_units(units3)
        t3.step(torch.from_numpy(tok3).to(dev))
        g3full = [t.cpu().numpy() for t in t3.full_units("g32")]
        for _ in range(2):                   # more steps: no barrier fault either
            t3.step(torch.from_numpy(tok3).to(dev))
        t3.check_faults()
        report["symm_status_odd"] = float(K.SymmWorkspace.status(reset=True))
        del t3

        stage(rank, "graph replay")
        # the multi-rank step as a CUDA graph (device-resident barrier epochs): five
        # steps eager against two eager + capture + replays, same tokens every step
        # (the l <= 1 plan: fused bf16-wire units; the l > 1 plan: fp32 accumulators,
        # NCCL-routed units wherever the route table sends them there)
        worst = 0.0
        for gplan, gtok in ((pplan, ptok), (plan, torch.from_numpy(tok).to(dev))):
            res = {}
            for graph in (False, True):
                tg = UnevenFSDPTrainer(arch, gplan, rank, comm_ag=cag, comm_rs=crs, device=dev,
                                       algo=K.ALGO_SYMM)
                tg.load_full_units(units)
                tg.graph = graph and tg.graph_eligible()
                for _ in range(5):
                    tg.step(gtok)
                tg.check_faults()
                if graph:
                    # (idle ranks and N > 4 stay eager: graph_eligible)
                    report[f"graph_active_{len(report)}"] = float(
                        tg.graph_active or not tg.graph_eligible())
                res[graph] = [t.cpu().numpy() for t in tg.full_units("p32")]
                del tg
            worst = max(worst, max(
                float(np.linalg.norm(a.astype(np.float64) - b) / max(np.linalg.norm(b), 1e-30))
                for a, b in zip(res[True], res[False])))
        report["graph_vs_eager"] = worst
        report["symm_status_graph"] = float(K.SymmWorkspace.status(reset=True))

        stage(rank, "fault injection")
        # fault injection: rank 0 enters a fused all-gather that no other rank joins
        # (shortened spin limit). Its barrier times out; the trainer's asynchronous
        # status check must then raise CollectiveFault on rank 0 after its next step
        # instead of training on that step's unsynchronised buffers.
        torch.cuda.synchronize()
        dist.barrier()
        K.set_symm_timeout_ms(300)
        if rank == 0:
            trs.symm.allgather_pack(torch.zeros(4, device=dev), "ub0", 0, [4] + [0] * (world - 1),
                                    [0] + [4] * (world - 1))
            torch.cuda.synchronize()
        K.set_symm_timeout_ms(10_000)
        if rank != 0:
            trs.symm.epoch[0] += 1      # every rank's AG channel epoch agrees again
        dist.barrier()
        raised = 0
        try:
            trs.step(torch.from_numpy(tok).to(dev))
            trs.check_faults()
        except K.CollectiveFault:
            raised = 1
        report["fault_raised"] = float(raised == (1 if rank == 0 else 0))
        K.SymmWorkspace.status(reset=True)
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        stage(rank, "saving")
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), loss=float(loss),
                 micro=np.array(micro), ratios=np.array(ratios),
                 report_keys=np.array(list(report.keys())),
                 report_vals=np.array(list(report.values()), dtype=np.float64),
                 loss_symm=float(loss_s),
                 **{f"g{u}": x for u, x in enumerate(g)}, **{f"p{u}": x for u, x in enumerate(p)},
                 **{f"gs{u}": x for u, x in enumerate(gs)},
                 **{f"ps{u}": x for u, x in enumerate(ps)},
                 **{f"gw{u}": x for u, x in enumerate(pair[True])},
                 **{f"gf{u}": x for u, x in enumerate(pair[False])},
                 pmicro=np.array(pmicro),
                 **{f"g3_{u}": x for u, x in enumerate(g3full)})
    finally:
        stage(rank, "teardown")
        cag.close()
        crs.close()
        dist.destroy_process_group()
        stage(rank, "done")


if __name__ == "__main__":
    main(sys.argv[1])
