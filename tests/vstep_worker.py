"""Worker of tests/test_virtual_step_gpu.py (one case per process):

  PYTORCH_CUDA_ALLOC_CONF=backend:cudaMallocAsync python tests/vstep_worker.py NAME N

Multi-rank train-step parity at the BASELINE layouts on ONE GPU.

N trainers (one per virtual rank, tests/vranks.py) run in N threads of one
process on one B200. Each has its own compute / all-gather / reduce-scatter
streams and its rank's view of one shared symmetric allocation, so the step
issues exactly the fused kernels it issues on N GPUs (peer and helper
routes; NVLS multicast needs real GPUs) and its ranks meet at the same
in-kernel barriers. The driver's 1-GPU test run thereby checks the N = 2, 4
and 8 step end to end against the CPU oracle.

Plans: the planner's bench plan of each config at N ranks
(configs.build_job: the shard layout of the real units from the plan's state
ratios, and each rank's l_i), with every microbatch m_i scaled down so the
fp32 CPU oracle finishes in seconds; the uneven Eq. 1 weights m_i / B, the
layered accumulation and the state layout are the plan's.

Bars (north_star): loss within 2e-2 relative; every unit's
reduced gradient within 2e-2 normwise of the oracle's Eq. 1 gradient
(gradcheck.py:30-46; sim.py:278-322), or within plain torch bf16 autograd's
own error where that exceeds 2e-2 (test_step_configs_gpu.grad_bar), and
element-wise within 5e-2 of the
unit's max|g|; post-AdamW master / moments within 1e-5 (max relative) of the
oracle's AdamW fed the reduced gradient; no barrier timeout.

Why a subprocess with the stream-ordered allocator: the CUDA programming
guide lists a device memory allocation and a page-locked host allocation as
implicit synchronisation points between streams. N ranks driven from threads
of one process share a device, so a caching-allocator cudaMalloc in a lagging
rank's thread would wait for a leading rank's fused kernel, which spins on
the lagging rank's matching kernel: deadlock until the barrier spin limit.
cudaMallocAsync allocations are stream-ordered and never synchronise.
(Separate processes on separate GPUs, the product setting, have no such
coupling.)
"""

import math
import os
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
for _p in (os.path.dirname(_HERE), _HERE):
    if _p not in sys.path:
        sys.path.insert(0, _p)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import model_oracle as MO  # noqa: E402
from oracle import step_oracle as SO  # noqa: E402
from oracle.tolerances import BF16_GRAD_RTOL, FP32_RTOL, max_rel, norm_rel  # noqa: E402
from paper_2411_01075_b200 import GpuAssignment, TrainPlan, assign_unit_shards  # noqa: E402
from paper_2411_01075_b200 import hetstep as K  # noqa: E402
from paper_2411_01075_b200.configs import build_job  # noqa: E402
from paper_2411_01075_b200.data import rank_tokens  # noqa: E402
from paper_2411_01075_b200.step import AdamWConfig, UnevenFSDPTrainer  # noqa: E402
from test_step_configs_gpu import grad_bar, torch_bf16_grads  # noqa: E402
from test_step_gpu import cpu_units  # noqa: E402
from vranks import VirtualGroup, VirtualRankGroup, VirtualSymmWorkspace, run_ranks  # noqa: E402


OPT = AdamWConfig()
OPT_D = dict(lr=OPT.lr, beta1=OPT.betas[0], beta2=OPT.betas[1], eps=OPT.eps,
             weight_decay=OPT.weight_decay)
ELEM_ABS = 5e-2


def scaled_plan(name: str, n: int, target_batch: int):
    """The bench plan at n ranks with microbatches scaled so B ~ target_batch."""
    job = build_job(name, n, measured=True)
    B = job.plan.total_batch
    k = max(1, math.ceil(B / target_batch))
    ratios = [a.state_ratio for a in job.plan.assignments]
    asg, tot = [], 0
    for a in job.plan.assignments:
        m = 0 if a.microbatch == 0 else max(1, a.microbatch // k)
        asg.append((m, a.num_microbatches if m else 0))
        tot += m * asg[-1][1]
    arch = job.arch
    model = arch.model_spec(tot)
    plan = TrainPlan(tuple(GpuAssignment(f"g{i}", m, l, m * l, r, 0.0, r * model.state_bytes)
                           for i, ((m, l), r) in enumerate(zip(asg, ratios))),
                     1.0, 1.0, 2.0 * arch.layers, True, assign_unit_shards(ratios, model))
    assert [list(r) for r in plan.unit_shards.shards] == \
        [list(r) for r in job.plan.unit_shards.shards]      # the bench layout itself
    return arch, plan


CASES = [("gpt2_small", 2), ("gpt2_small", 4), ("gpt2_small", 8), ("bert_large", 4),
         ("llama_1b3", 2), ("llama_1b3", 8)]


def run_case(cuda, name, n):
    arch, plan = scaled_plan(name, n, 8 if name != "llama_1b3" else 4)
    units = cpu_units(arch, seed=3)
    toks = [rank_tokens(plan, r, arch.seq, arch.vocab, seed=21, step=0) for r in range(n)]
    sms = torch.cuda.get_device_properties(cuda).multi_processor_count
    # both channels' kernels of every rank co-resident: 2 * n * ctas below the SM count
    vg = VirtualGroup(n, UnevenFSDPTrainer.symm_regions(arch), cuda,
                      ctas=max(1, min(32, (sms - 8) // (2 * n))))
    group = VirtualRankGroup(n)
    streams = [torch.cuda.Stream(device=cuda) for _ in range(n)]
    K.SymmWorkspace.status(reset=True)

    def build(r):
        with torch.cuda.stream(streams[r]):
            tr = UnevenFSDPTrainer(arch, plan, r, opt=OPT, device=cuda, algo=K.ALGO_SYMM,
                                   group=group, symm_workspace=VirtualSymmWorkspace(vg, r, group))
            tr.load_full_units(units)
            torch.cuda.current_stream().synchronize()
            return tr

    trs = run_ranks(n, build, group)
    assert all(t.route_check["ok"] for t in trs), [t.route_check for t in trs]
    assert all(r == "symm" for t in trs for r in t.ag_route + t.rs_route)
    p0 = [t.p32.clone() for t in trs]

    dtoks = [torch.from_numpy(t).to(cuda) for t in toks]
    torch.cuda.synchronize()

    def step(r):
        with torch.cuda.stream(streams[r]):
            loss = trs[r].step(dtoks[r])
            trs[r].check_faults()
            return float(loss)

    losses = run_ranks(n, step, group)
    torch.cuda.synchronize()
    assert K.SymmWorkspace.status(reset=True) == 0
    live = [(toks[r], (a.microbatch, a.num_microbatches))
            for r, a in enumerate(plan.assignments) if a.microbatch > 0]
    tb = torch_bf16_grads(arch, units, [t for t, _ in live], [mi for _, mi in live], cuda)
    gu, gr, ref_loss = MO.weighted_gradient(arch, units[:-1], units[-1], [t for t, _ in live],
                                            [mi for _, mi in live])
    assert abs(sum(losses) - ref_loss) <= BF16_GRAD_RTOL * abs(ref_loss)
    L = trs[0].L
    worst = 0.0
    for u, ref in enumerate(gu + [gr]):
        got = np.zeros(ref.numel(), np.float32)
        for r, t in enumerate(trs):
            off, cnt = t.L.local_range(u)
            o = L.offsets[u][r]
            got[o:o + cnt] = t.g32[off:off + cnt].cpu().numpy()
        want = ref.numpy()
        nr = norm_rel(got, want)
        worst = max(worst, nr)
        tb_err = norm_rel(tb[u], want)
        assert nr <= grad_bar(tb_err), f"{name} N={n} unit {u}: normwise {nr} (bf16 {tb_err})"
        ea = float(np.max(np.abs(got.astype(np.float64) - want)) / np.max(np.abs(want)))
        assert ea <= ELEM_ABS, f"{name} N={n} unit {u}: element abs {ea}"
    print(f"\n{name} N={n} plan {[(a.microbatch, a.num_microbatches) for a in plan.assignments]}"
          f" routes ag={set(trs[0].ag_policy)} rs={set(trs[0].rs_policy)}"
          f" wire16={sum(trs[0].wire16)}: worst normwise {worst:.2e}")
    for r, t in enumerate(trs):
        z = np.zeros(t.L.local_len, np.float32)
        rp, rm, rv = SO.adamw(p0[r].cpu().numpy(), t.g32.cpu().numpy(), z, z, step=1, **OPT_D)
        assert max_rel(t.p32.cpu().numpy(), rp) <= FP32_RTOL
        assert max_rel(t.m32.cpu().numpy(), rm) <= FP32_RTOL
        assert max_rel(t.v32.cpu().numpy(), rv) <= FP32_RTOL


if __name__ == "__main__":
    assert "cudaMallocAsync" in os.environ.get("PYTORCH_CUDA_ALLOC_CONF", ""), \
        "run with PYTORCH_CUDA_ALLOC_CONF=backend:cudaMallocAsync"
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    run_case(dev, sys.argv[1], int(sys.argv[2]))
    print("VSTEP_OK", flush=True)
