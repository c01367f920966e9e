"""Sharded checkpoint/resume keyed by UnitShardPlan, including re-sharding
onto a different plan (other ratios and rank count). CPU only."""
import torch

import fake_kernels
from paper_2411_01075_b200 import GpuAssignment, ModelSpec, TrainPlan, assign_unit_shards
from paper_2411_01075_b200 import step as S
from paper_2411_01075_b200.checkpoint import (STATE, checkpoint_plan, load_shards, load_trainer,
                                              save_shards, save_trainer)
from paper_2411_01075_b200.data import rank_tokens
from paper_2411_01075_b200.layout import RankLayout
from paper_2411_01075_b200.model import ARCHS


def _plan(arch, micro, ratios):
    B = sum(m * l for m, l in micro)
    model = ModelSpec(arch.layers, arch.unit_params, B)
    rows = tuple(GpuAssignment(f"g{i}", m, l, m * l, r, 0.0, r * model.state_bytes)
                 for i, ((m, l), r) in enumerate(zip(micro, ratios)))
    return TrainPlan(rows, 1.0, 1.0, 1.0, True, assign_unit_shards(ratios, model))


def _local_buffers(layout, fulls):
    out = {}
    for name in STATE:
        buf = torch.zeros(layout.local_len)
        for u in range(layout.blocks + 1):
            off, cnt = layout.local_range(u)
            o = layout.offsets[u][layout.rank]
            buf[off:off + cnt] = fulls[name][u][o:o + cnt]
        out[name] = buf
    return out


def test_reshard_onto_a_different_plan(tmp_path):
    arch = ARCHS["tiny_gpt"]
    g = torch.Generator().manual_seed(0)
    fulls = {n: [torch.randn(arch.unit_params, generator=g) for _ in range(arch.layers)] +
             [torch.randn(arch.root_params, generator=g)] for n in STATE}
    a = _plan(arch, [(2, 1), (1, 1)], [683 / 1024, 341 / 1024])
    for r in range(2):
        lay = RankLayout.from_plan(a, arch.unit_params, arch.root_params, r)
        save_shards(tmp_path, lay, _local_buffers(lay, fulls), step=7, plan=a)
    assert checkpoint_plan(tmp_path).unit_shards == a.unit_shards
    for b in (a, _plan(arch, [(1, 1)] * 3, [0.5, 0.0, 0.5]), _plan(arch, [(4, 1)], [1.0])):
        n = len(b.assignments)
        assembled = {name: [torch.zeros_like(t) for t in fulls[name]] for name in STATE}
        for r in range(n):
            lay = RankLayout.from_plan(b, arch.unit_params, arch.root_params, r)
            parts, step = load_shards(tmp_path, lay)
            assert step == 7
            for name in STATE:
                for u, t in enumerate(parts[name]):
                    o = lay.offsets[u][r]
                    assembled[name][u][o:o + t.numel()] = t
        for name in STATE:
            for x, y in zip(assembled[name], fulls[name]):
                assert torch.equal(x, y)


def test_trainer_resume_is_exact(tmp_path, monkeypatch):
    monkeypatch.setattr(S, "K", fake_kernels)
    arch = ARCHS["tiny_gpt"]
    plan = _plan(arch, [(2, 1)], [1.0])
    t1 = S.UnevenFSDPTrainer(arch, plan, 0, device=torch.device("cpu"))
    t1.init_params(3)
    tok = lambda s: torch.from_numpy(rank_tokens(plan, 0, arch.seq, arch.vocab, 1, s))  # noqa
    t1.step(tok(0))
    save_trainer(t1, tmp_path)
    t2 = S.UnevenFSDPTrainer(arch, plan, 0, device=torch.device("cpu"))
    assert load_trainer(t2, tmp_path) == 1
    for name in STATE + ("p16",):
        assert torch.equal(getattr(t1, name), getattr(t2, name))
    l1, l2 = t1.step(tok(1)), t2.step(tok(1))
    assert torch.equal(l1, l2) and torch.equal(t1.p32, t2.p32)
