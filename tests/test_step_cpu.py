"""Host-side logic of the step driver on CPU: schedule, layout, autograd
plumbing and the Eq. 1 weighting, with the CUDA kernels replaced by the
oracle-backed test double (tests/fake_kernels.py). N=1 here; world_size 2
over gloo in tests/test_multirank_cpu.py."""
import pytest
import torch

import fake_kernels
from oracle import model_oracle as MO
from paper_2411_01075_b200 import GpuAssignment, ModelSpec, TrainPlan, assign_unit_shards
from paper_2411_01075_b200 import step as S
from paper_2411_01075_b200.data import rank_tokens
from paper_2411_01075_b200.model import ARCHS, init_flat


@pytest.fixture
def fake(monkeypatch):
    monkeypatch.setattr(S, "K", fake_kernels)
    fake_kernels.calls.clear()
    return fake_kernels


def _plan(arch, m, l):
    model = ModelSpec(arch.layers, arch.unit_params, m * l)
    return TrainPlan((GpuAssignment("g0", m, l, m * l, 1.0, 0.0, float(model.state_bytes)),),
                     1.0, 1.0, 2.0 * arch.layers, False, assign_unit_shards([1.0], model))


def _units(arch):
    out = []
    for u in range(arch.layers + 1):
        g = torch.Generator().manual_seed(u)
        out.append(init_flat(arch.root_layout() if u == arch.layers else arch.unit_layout(), g,
                             "cpu"))
    return out


@pytest.mark.parametrize("m,l", [(2, 1), (1, 3)])
def test_single_rank_step_gradients(fake, m, l):
    arch = ARCHS["tiny_gpt"]
    plan = _plan(arch, m, l)
    units = _units(arch)
    tr = S.UnevenFSDPTrainer(arch, plan, 0, device=torch.device("cpu"))
    tr.load_full_units(units)
    tok = rank_tokens(plan, 0, arch.seq, arch.vocab, seed=5, step=0)
    loss = float(tr.step(torch.from_numpy(tok)))
    gu, gr, ref = MO.weighted_gradient(arch, units[:-1], units[-1], [tok], [(m, l)])
    assert abs(loss - ref) <= 2e-2 * abs(ref)
    for u, g in enumerate(gu + [gr]):
        off, cnt = tr.L.local_range(u)
        got = tr.g32[off:off + cnt].double()
        assert float((got - g.double()).norm() / g.double().norm()) <= 2e-2
    # one accumulate per (unit, microbatch) + head and embedding passes, one AdamW
    n_acc = fake.calls.count("accumulate")
    # l=1, one rank: one grouped launch; l>1: microbatches folded in groups of
    # tr.acc_microbatches per unit
    unit_launches = 1 if l == 1 else arch.layers * -(-l // tr.acc_microbatches)
    assert n_acc == unit_launches + l            # units + head; embedding is fused
    assert fake.calls.count("embedding_grad") == l
    assert fake.calls.count("adamw") == 1
    assert "allgather" not in fake.calls and "reduce_scatter" not in fake.calls


def test_head_row_chunks_match_whole_microbatch(fake):
    """head_chunk (a memory-capped rank's head in row chunks, each with its
    share of the gradient) gives the whole-microbatch step's loss and
    gradients to fp32 rounding."""
    arch = ARCHS["tiny_gpt"]
    plan = _plan(arch, 3, 1)
    units = _units(arch)
    tok = torch.from_numpy(rank_tokens(plan, 0, arch.seq, arch.vocab, seed=6, step=0))
    out = {}
    for chunk in (None, 2):
        tr = S.UnevenFSDPTrainer(arch, plan, 0, device=torch.device("cpu"))
        tr.load_full_units(units)
        tr.head_chunk = chunk
        fake.calls.clear()
        out[chunk] = (float(tr.step(tok)), tr.g32.clone(), fake.calls.count("accumulate"))
    assert abs(out[2][0] - out[None][0]) <= 2e-2 * abs(out[None][0])
    g0, g2 = out[None][1].double(), out[2][1].double()
    assert float((g2 - g0).norm() / g0.norm()) <= 2e-2
    assert out[2][2] == out[None][2] + 1          # two head chunks: one more root accumulate
