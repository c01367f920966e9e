"""End-to-end parity of the B200 train step on one GPU against the CPU
oracle (oracle/model_oracle.py, torch CPU fp32, independent model code).

Tolerances (north_star): gradients computed from bf16 activations/params are
compared normwise — ||g_gpu - g_ref|| / ||g_ref|| <= 2e-2 per unit; the
optimizer and layout arithmetic downstream of those gradients is compared
at max relative error 1e-5 against the oracle fed the GPU's own reduced
gradients; the bf16 shadow is bit-exact.
"""
import numpy as np
import pytest
import torch

from oracle import model_oracle as MO
from oracle import step_oracle as SO
from oracle.tolerances import max_rel as _mrel
from oracle.tolerances import norm_rel as _nrel
from paper_2411_01075_b200 import GpuAssignment, ModelSpec, TrainPlan, assign_unit_shards
from paper_2411_01075_b200.data import rank_tokens
from paper_2411_01075_b200.model import ARCHS, init_flat
from paper_2411_01075_b200.step import AdamWConfig, UnevenFSDPTrainer

pytestmark = pytest.mark.gpu

OPT = AdamWConfig()
OPT_D = dict(lr=OPT.lr, beta1=OPT.betas[0], beta2=OPT.betas[1], eps=OPT.eps,
             weight_decay=OPT.weight_decay)


def one_gpu_plan(arch, m, l):
    model = ModelSpec(layers=arch.layers, params_per_layer=arch.unit_params, global_batch=m * l)
    a = GpuAssignment("g0", m, l, m * l, 1.0, 0.0, float(model.state_bytes))
    return TrainPlan((a,), 1.0, 1.0, arch.layers * 2.0, False, assign_unit_shards([1.0], model))


def cpu_units(arch, seed=0):
    units = []
    for u in range(arch.layers + 1):
        g = torch.Generator().manual_seed(seed * 100003 + u)
        lay = arch.root_layout() if u == arch.layers else arch.unit_layout()
        units.append(init_flat(lay, g, "cpu"))
    return units


@pytest.mark.parametrize("m,l", [(4, 1), (2, 3)])
def test_single_gpu_step_matches_cpu_oracle(cuda, m, l):
    arch = ARCHS["tiny_gpt"]
    plan = one_gpu_plan(arch, m, l)
    units = cpu_units(arch)
    tr = UnevenFSDPTrainer(arch, plan, 0, opt=OPT, device=cuda)
    tr.load_full_units(units)
    p0 = tr.p32.clone()
    tok = rank_tokens(plan, 0, arch.seq, arch.vocab, seed=1234, step=0)
    loss = tr.step(torch.from_numpy(tok).to(cuda))
    torch.cuda.synchronize()

    # model-level: weighted full-batch gradient vs CPU fp32 (bf16 tolerance)
    gu, gr, ref_loss = MO.weighted_gradient(arch, units[:-1], units[-1], [tok], [(m, l)])
    assert abs(float(loss) - ref_loss) / abs(ref_loss) <= 2e-2
    for u, ref in enumerate(gu + [gr]):
        off, cnt = tr.L.local_range(u)
        got = tr.g32[off:off + cnt].cpu().numpy()
        assert _nrel(got, ref.numpy()) <= 2e-2, f"unit {u}"

    # shard math downstream of the GPU's own reduced gradients: 1e-5 / bit-exact
    rp, rm, rv = SO.adamw(p0.cpu().numpy(), tr.g32.cpu().numpy(),
                          np.zeros(tr.L.local_len, np.float32), np.zeros(tr.L.local_len, np.float32),
                          step=1, **OPT_D)
    assert _mrel(tr.p32.cpu().numpy(), rp) <= 1e-5
    assert _mrel(tr.m32.cpu().numpy(), rm) <= 1e-5
    assert _mrel(tr.v32.cpu().numpy(), rv) <= 1e-5
    shadow = tr.p16.view(torch.int16).cpu().numpy().view(np.uint16)
    assert np.array_equal(shadow, SO.pack(tr.p32.cpu().numpy()))


def test_loss_decreases_over_steps(cuda):
    arch = ARCHS["tiny_gpt"]
    plan = one_gpu_plan(arch, 4, 2)
    tr = UnevenFSDPTrainer(arch, plan, 0, opt=OPT, device=cuda)
    tr.init_params(seed=3)
    tok = torch.from_numpy(rank_tokens(plan, 0, arch.seq, arch.vocab, seed=7, step=0)).to(cuda)
    losses = [float(tr.step(tok)) for _ in range(8)]   # same batch: must overfit
    assert losses[-1] < losses[0] - 0.05, losses


def test_checkpoint_resume_on_gpu(cuda, tmp_path):
    from paper_2411_01075_b200.checkpoint import load_trainer, save_trainer
    arch = ARCHS["tiny_gpt"]
    plan = one_gpu_plan(arch, 2, 2)
    a = UnevenFSDPTrainer(arch, plan, 0, opt=OPT, device=cuda)
    a.init_params(seed=5)
    tok = [torch.from_numpy(rank_tokens(plan, 0, arch.seq, arch.vocab, seed=2, step=s)).to(cuda)
           for s in range(2)]
    a.step(tok[0])
    save_trainer(a, tmp_path)
    b = UnevenFSDPTrainer(arch, plan, 0, opt=OPT, device=cuda)
    assert load_trainer(b, tmp_path) == 1
    for name in ("p32", "m32", "v32", "p16"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name
    la, lb = a.step(tok[1]), b.step(tok[1])
    torch.cuda.synchronize()
    # the resumed step matches (attention backward may reduce in a different order)
    assert abs(float(la) - float(lb)) <= 1e-6 * abs(float(la))
    assert _nrel(b.p32.cpu().numpy(), a.p32.cpu().numpy()) <= 1e-5


@pytest.mark.parametrize("schedule", ["reference", "checkpoints"])
def test_activation_offload_matches_and_saves_memory(cuda, schedule):
    """Checkpoint offload leaves the step's math
    unchanged, is lint-clean against the simulator's offload rules, and cuts
    the resident boundary activations."""
    arch = ARCHS["gpt2_small"]
    plan = one_gpu_plan(arch, 4, 4)
    tok = torch.from_numpy(rank_tokens(plan, 0, arch.seq, arch.vocab, seed=3, step=0)).to(cuda)
    res = {}
    torch.use_deterministic_algorithms(True)   # deterministic cuDNN attention backward
    try:
        _offload_runs(arch, plan, tok, cuda, res, schedule)
    finally:
        torch.use_deterministic_algorithms(False)
    if schedule == "reference":
        # l_i = 4: the full reference schedule, activation gradients included
        assert {"offload_act", "prefetch_act", "offload_grad", "prefetch_grad"} <= res[True][3]
    else:
        # checkpoints only: the in-flight boundary tensors stay on the GPU
        assert {"offload_act", "prefetch_act"} <= res[True][3]
        assert not {"offload_grad", "prefetch_grad"} & res[True][3]
    assert res[True][0] == res[False][0]
    assert torch.equal(res[True][1], res[False][1])       # offload moves bytes, not math
    # 12 units x 4 microbatches x [4, 512, 768] bf16 checkpoints = 151 MB resident without
    # offload; with it a few boundary tensors stay on the GPU
    assert res[True][2] < res[False][2] - 120e6, (res[True][2], res[False][2])


def _offload_runs(arch, plan, tok, cuda, res, schedule="reference"):
    from paper_2411_01075_b200.trace import StepTracer, lint_measured_trace
    for off in (False, True):
        tr = UnevenFSDPTrainer(arch, plan, 0, opt=OPT, device=cuda, offload_activations=off,
                               offload_schedule=schedule)
        tr.init_params(seed=1)
        tr.step(tok)
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats(cuda)
        base = torch.cuda.memory_allocated(cuda)
        tr.tracer = StepTracer("g0")
        loss = tr.step(tok)
        ev = tr.tracer.collect()
        peak = torch.cuda.max_memory_allocated(cuda) - base
        assert lint_measured_trace(ev, arch.layers) == [], off
        res[off] = (float(loss), tr.p32.clone(), peak, {e.kind for e in ev})
        del tr


def test_llama_unit_step_matches_cpu_oracle(cuda):
    """Llama-style units (fused RMSNorm, in-place RoPE, SwiGLU) against the
    independent fp32 CPU model oracle."""
    from paper_2411_01075_b200.model import ArchSpec
    arch = ArchSpec("tiny_llama", "llama", d=256, layers=2, heads=2, ffn=512, vocab=4096, seq=128)
    plan = one_gpu_plan(arch, 2, 2)
    units = cpu_units(arch, seed=4)
    tr = UnevenFSDPTrainer(arch, plan, 0, opt=OPT, device=cuda)
    tr.load_full_units(units)
    tok = rank_tokens(plan, 0, arch.seq, arch.vocab, seed=9, step=0)
    loss = tr.step(torch.from_numpy(tok).to(cuda))
    torch.cuda.synchronize()
    gu, gr, ref_loss = MO.weighted_gradient(arch, units[:-1], units[-1], [tok], [(2, 2)])
    assert abs(float(loss) - ref_loss) / abs(ref_loss) <= 2e-2
    for u, ref in enumerate(gu + [gr]):
        off, cnt = tr.L.local_range(u)
        assert _nrel(tr.g32[off:off + cnt].cpu().numpy(), ref.numpy()) <= 2e-2, f"unit {u}"


@pytest.mark.parametrize("m,l", [(4, 1), (2, 3)])
def test_cuda_graph_step_matches_eager(cuda, m, l):
    """The N=1 step replayed as one CUDA graph (tokens copied into the captured
    input, AdamW coefficients staged per replay through het_adamw_devcoef) is
    bitwise the eager step, step after step, and counts its owned launches."""
    from paper_2411_01075_b200 import hetstep as K
    arch = ARCHS["gpt2_small"]
    plan = one_gpu_plan(arch, m, l)
    toks = [torch.from_numpy(rank_tokens(plan, 0, arch.seq, arch.vocab, seed=4, step=s)).to(cuda)
            for s in range(6)]
    res = {}
    torch.use_deterministic_algorithms(True)
    try:
        for graph in (False, True):
            tr = UnevenFSDPTrainer(arch, plan, 0, opt=OPT, device=cuda)
            tr.init_params(seed=2)
            tr.graph = graph
            n0 = K.LAUNCHES
            losses = [float(tr.step(t)) for t in toks]
            torch.cuda.synchronize()
            res[graph] = (losses, tr.p32.clone(), tr.v32.clone(), K.LAUNCHES - n0, tr.steps,
                          tr.graph_active)
            del tr
    finally:
        torch.use_deterministic_algorithms(False)
    assert res[True][5] and not res[False][5]
    assert res[True][0] == res[False][0]
    assert torch.equal(res[True][1], res[False][1])
    assert torch.equal(res[True][2], res[False][2])
    assert res[True][3] == res[False][3] and res[True][4] == res[False][4] == 6


def test_head_row_chunks_on_gpu(cuda):
    """A memory-capped rank's head in row chunks (head_chunk) against the whole
    microbatch: fp32 loss to 1e-5, reduced gradients within the bf16 bar."""
    arch = ARCHS["gpt2_small"]
    plan = one_gpu_plan(arch, 4, 2)
    tok = torch.from_numpy(rank_tokens(plan, 0, arch.seq, arch.vocab, seed=8, step=0)).to(cuda)
    out = {}
    for chunk in (None, 1):
        tr = UnevenFSDPTrainer(arch, plan, 0, opt=OPT, device=cuda)
        tr.init_params(seed=3)
        tr.head_chunk = chunk
        loss = float(tr.step(tok))
        torch.cuda.synchronize()
        out[chunk] = (loss, tr.g32.double().clone())
        del tr
    assert abs(out[1][0] - out[None][0]) <= 1e-5 * abs(out[None][0])
    assert float((out[1][1] - out[None][1]).norm() / out[None][1].norm()) <= 2e-2


def test_offload_residency_contract(cuda):
    """The reference's residency contract on a MEASURED step (sim.py ledger rules,
    trace.boundary_residency; test_acceptance.py:157-186): with l = 4 the
    schedule keeps l + 1 = 5 boundary items resident without offload and 2 with
    the reference offload schedule."""
    from paper_2411_01075_b200.trace import StepTracer, boundary_residency, lint_measured_trace
    arch = ARCHS["gpt2_small"]
    plan = one_gpu_plan(arch, 4, 4)
    tok = torch.from_numpy(rank_tokens(plan, 0, arch.seq, arch.vocab, seed=5, step=0)).to(cuda)
    peaks = {}
    for off in (False, True):
        tr = UnevenFSDPTrainer(arch, plan, 0, opt=OPT, device=cuda, offload_activations=off,
                               offload_schedule="reference")
        tr.init_params(seed=1)
        tr.keep_last_graph = False
        tr.step(tok)
        tr.tracer = StepTracer("g0")
        tr.step(tok)
        ev = tr.tracer.collect()
        assert lint_measured_trace(ev, arch.layers) == []
        peaks[off] = boundary_residency(ev, arch.layers)["g0"]
        del tr
    assert peaks[False] == 4 + 1, peaks
    assert peaks[True] == 2, peaks
