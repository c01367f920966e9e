"""Pin the CPU oracle before trusting it (CPU only).

* Eq. 1 weighting of the step (per-rank w_i = m_i/B on l_i accumulated
  microbatch-mean gradients, SUM reduce-scatter) against the reference's own
  weighted_combine / full_batch_mean outputs (tests/golden/weighted_combine.json).
* AdamW against torch.optim.AdamW on CPU (the reference has no optimizer
  code: "parity unpinned" by the reference, pinned to torch here).
* bf16 packing against torch's fp32->bf16 conversion (RNE), bit-exact.
* all-gather / reduce-scatter restatements on the reference's shard goldens.
"""
import json
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2411_01075_b200 as H
from oracle import step_oracle as O
from oracle.tolerances import FP32_RTOL, max_rel

GOLD = Path(__file__).resolve().parent / "golden"


def test_weighted_combine_matches_reference_golden_exactly():
    g = json.loads((GOLD / "weighted_combine.json").read_text())
    for c in g["cases"]:
        got = H.weighted_combine([np.array(m) for m in c["means"]], c["batches"])
        assert got.tolist() == c["weighted"]
    rep = H.run_check(fixtures=200, seed=0)
    assert rep.max_rel_error == g["run_check_200_seed0"]["max_rel_error"]
    assert rep.max_unweighted_rel_error == g["run_check_200_seed0"]["max_unweighted_rel_error"]


@pytest.mark.parametrize("seed", range(5))
def test_step_weighting_reproduces_reference_eq1(seed):
    """Split each golden fixture's per-GPU batch b_i into l_i microbatches of
    m_i, run the oracle's accumulate(w=m_i/B) + reduce-scatter, and compare
    with the reference formula (weighted_combine) applied to the per-GPU means
    those microbatches imply: equal to fp32 precision (1e-5)."""
    g = json.loads((GOLD / "weighted_combine.json").read_text())
    rng = np.random.default_rng(seed)
    for c in g["cases"][seed::5]:
        b = c["batches"]
        B = sum(b)
        dim = len(c["means"][0])
        accs, gpu_means = [], []
        for bi, mean in zip(b, c["means"]):
            divs = [d for d in range(1, bi + 1) if bi % d == 0]
            m = int(rng.choice(divs))
            l = bi // m
            # l distinct microbatch means around the GPU mean
            mb = np.asarray(mean)[None, :] + 0.1 * rng.standard_normal((l, dim))
            q = [O.bf16_bits(mb[k].astype(np.float32)) for k in range(l)]
            acc = None
            for k in range(l):
                acc = O.accumulate(acc, q[k], k == 0, m / B)
            accs.append(acc)
            # the GPU's per-sample mean gradient implied by these microbatch means
            gpu_means.append(np.mean([O.bf16_to_f32(x).astype(np.float64) for x in q], axis=0))
        counts = [dim // 2, dim - dim // 2]
        red = np.concatenate(O.reduce_scatter(accs, counts, [0, counts[0]]))
        assert max_rel(red, H.weighted_combine(gpu_means, b)) <= FP32_RTOL


def test_step_weighting_exact_without_noise():
    """One microbatch per GPU (m_i = b_i, l_i = 1): the oracle's scale-cast +
    SUM reduce-scatter equals the reference formula on the bf16-rounded
    means to fp32 precision."""
    g = json.loads((GOLD / "weighted_combine.json").read_text())
    for c in g["cases"]:
        b, B = c["batches"], sum(c["batches"])
        accs, rounded = [], []
        for bi, mean in zip(b, c["means"]):
            q = O.bf16_bits(np.asarray(mean, np.float32))
            rounded.append(O.bf16_to_f32(q).astype(np.float64))
            accs.append(O.accumulate(None, q, True, bi / B))
        red = O.reduce_scatter(accs, [len(accs[0])], [0])[0]
        assert max_rel(red, H.weighted_combine(rounded, b)) <= FP32_RTOL


def test_bf16_wire_reduce_scatter_is_eq1():
    """The bf16-wire reduce-scatter (weights and cast inside the RS) equals the
    fp32-accumulate route bit for bit (same fl(w g) products, same rank-order
    sums) and the reference formula to fp32 precision."""
    g = json.loads((GOLD / "weighted_combine.json").read_text())
    for c in g["cases"]:
        b, B = c["batches"], sum(c["batches"])
        bits = [O.bf16_bits(np.asarray(m, np.float32)) for m in c["means"]]
        w = [bi / B for bi in b]
        dim = len(c["means"][0])
        counts = [dim // 2, dim - dim // 2]
        offs = [0, counts[0]]
        got = np.concatenate(O.reduce_scatter_bf16(bits, w, counts, offs))
        accs = [O.accumulate(None, q, True, wi) for q, wi in zip(bits, w)]
        fp32 = np.zeros(dim, np.float32)
        for a in accs:
            fp32 = fp32 + a
        assert np.array_equal(got, fp32)
        ref = H.weighted_combine([O.bf16_to_f32(q).astype(np.float64) for q in bits], b)
        assert max_rel(got, ref) <= FP32_RTOL


def test_rs_scale_is_eq1():
    plan = H.TrainPlan(tuple(H.GpuAssignment(f"g{i}", m, l, m * l, r, 0.0, 0.0)
                             for i, (m, l, r) in enumerate([(3, 2, 0.5), (1, 4, 0.5), (0, 0, 0.0)])),
                       1.0, 1.0, 2.0, True)
    assert H.rs_scale(plan) == [3 / 10, 1 / 10, 0.0]


@pytest.mark.parametrize("step", [1, 2, 10])
def test_adamw_oracle_matches_torch(step):
    n = 50_000
    g = torch.Generator().manual_seed(step)
    p = torch.randn(n, generator=g) * 0.02
    ref = torch.nn.Parameter(p.clone())
    opt = torch.optim.AdamW([ref], lr=1e-3, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1,
                            foreach=False)
    pp, m, v = p.numpy().copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)
    for s in range(1, step + 1):
        grad = torch.randn(n, generator=g) * 1e-3
        ref.grad = grad
        opt.step()
        pp, m, v = O.adamw(pp, grad.numpy(), m, v, lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8,
                           weight_decay=0.1, step=s)
    assert max_rel(pp, ref.detach().numpy()) <= FP32_RTOL
    st = opt.state[ref]
    assert max_rel(m, st["exp_avg"].numpy()) <= FP32_RTOL
    assert max_rel(v, st["exp_avg_sq"].numpy()) <= FP32_RTOL


def test_bf16_pack_matches_torch_rne():
    x = np.concatenate([np.random.default_rng(0).standard_normal(100_000).astype(np.float32) * 7,
                        np.array([0.0, -0.0, np.inf, -np.inf, 1e-40, 3.0e38, 1.00390625,
                                  1.01171875], np.float32)])
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(O.pack(x), ref)


def test_collective_restatements_on_shard_goldens():
    g = json.loads((GOLD / "sharding.json").read_text())
    rng = np.random.default_rng(3)
    for c in g["cases"][:40]:
        U = c["unit_params"]
        if U > 200_000:
            continue
        for counts, offs in zip(c["shards"][:2], c["offsets"][:2]):
            full = rng.standard_normal(U).astype(np.float32)
            sends = [O.pack(full[o:o + k]) for k, o in zip(counts, offs)]
            assert np.array_equal(O.allgather(sends, counts, offs), O.pack(full))
            srcs = [rng.standard_normal(U).astype(np.float32) for _ in counts]
            parts = O.reduce_scatter(srcs, counts, offs)
            assert [p.size for p in parts] == counts
            assert max_rel(np.concatenate(parts), np.sum(np.stack(srcs).astype(np.float64), 0)) \
                <= FP32_RTOL
