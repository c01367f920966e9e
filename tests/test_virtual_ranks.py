"""Parity of the fused uneven collectives at N = 2, 4 and 8 ranks on ONE GPU.

The virtual-rank harness (tests/vranks.py) runs N ranks, as one cooperative launch, of
het_symm_allgather_pack / het_symm_reduce_scatter / het_symm_reduce_scatter_bf16
over N copies of the symmetric buffer in one allocation, so the 1-GPU test
run proves the rank-count specialisations (NR = 2, 4, 8), the peer and relay
all-gathers, the peer reduce-scatter and the bf16-wire reduce-scatter
against the oracle, on:

  * the shard shapes of tests/mgpu_worker.py (even, ragged, single-owner at
    either end, the 3,571,623-param misaligned GPT-2 shard, random), each at
    a 16-byte-aligned and an odd unit offset;
  * every unit shape (blocks + root) of the trainer's layout for the
    planner's gpt2_small / bert_large / llama_1b3 bench plans at N = 8
    (reference sharding.py:89-95 offsets, gradcheck.py:30-46 weights).

Every route runs: AUTO / PEER (plain push / pull), RELAY (pair relay
all-gather) and HELPERS (light ranks relay or reduce pieces of the heavy
owners' ranges, hetstep_symm.cu helper_plan) for all three collectives.

Bars: all-gather bit-exact vs oracle.allgather of the packed ranges; fp32
reduce-scatter bit-exact vs the rank-ordered fp32 sum (the peer route's
order) and within 1e-5 of oracle.reduce_scatter (fp64 sum); bf16-wire
reduce-scatter bit-exact vs oracle.reduce_scatter_bf16. het_symm_status
must stay 0 (no barrier timed out).

All N ranks of a collective run as ONE cooperative launch (het_symm_virtual),
so every CTA that waits on another is co-resident by construction. The
multicast (NVLS) route needs N real GPUs; tests/test_multigpu.py covers it.
"""
from __future__ import annotations

import time

import numpy as np
import pytest
import torch

from oracle import step_oracle as O
from oracle.tolerances import FP32_RTOL, max_rel
from paper_2411_01075_b200 import hetstep as K
from vranks import VirtualGroup

pytestmark = pytest.mark.gpu


def shard_cases(n: int) -> list[list[int]]:
    cases = [[1000] * n, [1001] * (n - 1) + [999], [4096 * 7 + 3] + [0] * (n - 1),
             [0] * (n - 1) + [12345], [3_571_623] + [3_516_249] * (n - 1)]
    rng = np.random.default_rng(n)
    cases.append([int(x) for x in rng.integers(0, 50_000, size=n)])
    # 2:1 skew (the relay's pairing), geometric skew
    cases.append([2000 * (2 if j % 2 == 0 else 1) + j for j in range(n)])
    cases.append([max(1, 40_000 >> j) for j in range(n)])
    return [c for c in cases if sum(c) > 0]


def _offsets(c):
    return [int(sum(c[:j])) for j in range(len(c))]


def planner_shapes(name: str, n: int) -> list[tuple[list[int], list[int]]]:
    """Distinct (counts, offsets) of every unit (blocks + root) the trainer
    uses for the bench plan of `name` at n ranks."""
    from paper_2411_01075_b200.configs import build_job
    from paper_2411_01075_b200.layout import RankLayout
    job = build_job(name, n, measured=True)
    lay = RankLayout.from_plan(job.plan, job.arch.unit_params, job.arch.root_params, 0)
    seen, out = set(), []
    for c, o in zip(lay.counts, lay.offsets):
        if tuple(c) not in seen:
            seen.add(tuple(c))
            out.append((list(c), list(o)))
    return out


def _rank_srcs(total: int, n: int, seed: int) -> list[np.ndarray]:
    base = np.random.default_rng(seed).standard_normal(total, dtype=np.float32)
    return [np.roll(base, 7919 * r) * np.float32(1 + 0.25 * r) for r in range(n)]


def check_allgather(vg: VirtualGroup, counts, offs, policy, shift, seed):
    n, total = vg.n, sum(counts)
    full = np.random.default_rng(seed).standard_normal(total, dtype=np.float32)
    dev = vg.device
    srcs = [torch.from_numpy(full[offs[r]:offs[r] + counts[r]]).to(dev) for r in range(n)]
    for r in range(n):
        vg.view(r, "unit").fill_(float("nan"))
    vg.allgather_pack(srcs, "unit", 8 * shift, counts, offs, policy=policy)
    want = O.allgather([O.pack(full[o:o + c]) for c, o in zip(counts, offs)], counts, offs)
    for r in range(n):
        got = vg.view(r, "unit")[8 * shift:8 * shift + total].view(torch.int16).cpu().numpy()
        assert np.array_equal(got.view(np.uint16), want), \
            f"AG n={n} policy={policy} shift={shift} rank {r} counts={counts}"


def check_reduce_scatter(vg: VirtualGroup, counts, offs, shift, seed, policy=K.SYMM_AUTO):
    n, total, dev = vg.n, sum(counts), vg.device
    srcs = _rank_srcs(total, n, seed)
    for r in range(n):
        vg.view(r, "acc")[4 * shift:4 * shift + total].copy_(torch.from_numpy(srcs[r]))
    outs = [torch.full((counts[r],), float("nan"), device=dev) for r in range(n)]
    vg.reduce_scatter("acc", 4 * shift, outs, counts, offs, policy=policy)
    ordered = srcs[0].copy()
    for r in range(1, n):
        ordered = ordered + srcs[r]          # fp32, rank order (the peer route)
    want = O.reduce_scatter(srcs, counts, offs)
    for r in range(n):
        got = outs[r].cpu().numpy()
        lo = offs[r]
        assert np.array_equal(got, ordered[lo:lo + counts[r]]), \
            f"RS n={n} shift={shift} policy={policy} rank {r} not the rank-ordered fp32 sum"
        if counts[r]:
            assert max_rel(got, want[r]) <= FP32_RTOL


def check_reduce_scatter_bf16(vg: VirtualGroup, counts, offs, shift, seed, weights,
                              policy=K.SYMM_AUTO):
    n, total, dev = vg.n, sum(counts), vg.device
    bits = [O.pack(s) for s in _rank_srcs(total, n, seed)]
    for r in range(n):
        vg.view(r, "g16")[8 * shift:8 * shift + total].copy_(
            torch.from_numpy(bits[r].view(np.int16)).view(torch.bfloat16))
    outs = [torch.full((counts[r],), float("nan"), device=dev) for r in range(n)]
    vg.reduce_scatter_bf16("g16", 8 * shift, outs, counts, offs, weights, policy=policy,
                           stage="acc" if policy == K.SYMM_HELPERS else None)
    want = O.reduce_scatter_bf16(bits, weights, counts, offs)
    for r in range(n):
        assert np.array_equal(outs[r].cpu().numpy(), want[r]), \
            f"bf16-wire RS n={n} shift={shift} policy={policy} rank {r} counts={counts}"


def _weights(n: int) -> list[float]:
    # uneven Eq. 1 weights m_j / B, with one idle rank (w = 0) for n > 2
    m = [3 + (j % 3) for j in range(n)]
    if n > 2:
        m[1] = 0
    return [x / sum(m) for x in m]


@pytest.fixture(autouse=True)
def _status_clean(cuda):
    K.SymmWorkspace.status(reset=True)
    yield
    assert K.SymmWorkspace.status(reset=True) == 0, "a symmetric barrier timed out"


@pytest.mark.parametrize("n", [2, 4, 8])
def test_virtual_ranks_shard_cases(cuda, n):
    cases = shard_cases(n)
    maxu = max(sum(c) for c in cases) + 64
    vg = VirtualGroup(n, [("unit", maxu, torch.bfloat16), ("acc", maxu, torch.float32),
                          ("g16", maxu, torch.bfloat16)], cuda)
    for ci, counts in enumerate(cases):
        offs = _offsets(counts)
        for shift in (0, 3):
            for policy in (K.SYMM_AUTO, K.SYMM_PEER, K.SYMM_RELAY, K.SYMM_HELPERS):
                check_allgather(vg, counts, offs, policy, shift, seed=ci)
            for policy in (K.SYMM_AUTO, K.SYMM_HELPERS):
                check_reduce_scatter(vg, counts, offs, shift, 100 + ci, policy)
                check_reduce_scatter_bf16(vg, counts, offs, shift, 200 + ci, _weights(n), policy)


@pytest.mark.parametrize("name", ["gpt2_small", "bert_large", "llama_1b3"])
def test_virtual_ranks_planner_shapes_n8(cuda, name):
    n = 8
    shapes = planner_shapes(name, n)
    maxu = max(sum(c) for c, _ in shapes) + 64
    vg = VirtualGroup(n, [("unit", maxu, torch.bfloat16), ("acc", maxu, torch.float32),
                          ("g16", maxu, torch.bfloat16)], cuda)
    policies = {K.SYMM_AUTO, K.SYMM_RELAY, K.SYMM_HELPERS, K.ag_symm_policy(shapes[0][0], n)}
    for si, (counts, offs) in enumerate(shapes):
        for policy in sorted(policies):
            check_allgather(vg, counts, offs, policy, 0, seed=si)
        for policy in (K.SYMM_AUTO, K.SYMM_HELPERS):
            check_reduce_scatter(vg, counts, offs, 0, 300 + si, policy)
            check_reduce_scatter_bf16(vg, counts, offs, 0, 400 + si, _weights(n), policy)


@pytest.mark.parametrize("n", [2, 4, 8])
def test_device_epochs(cuda, n):
    """Device-resident barrier epochs (the CUDA-graph replay of a multi-rank
    step): every rank's base seeded with het_symm_epoch_set, launches passing
    EPOCH_DEVICE | offset, the base advanced with het_symm_epoch_add between
    "replays". The collectives stay exact, no barrier times out, and the start
    barrier's slots hold base + offset (the epoch the kernel resolved), not the
    raw argument."""
    counts = [3_571_623 // 64 + 5 * j for j in range(n)]
    offs = _offsets(counts)
    vg = VirtualGroup(n, [("unit", sum(counts) + 64, torch.bfloat16),
                          ("acc", sum(counts) + 64, torch.float32),
                          ("g16", sum(counts) + 64, torch.bfloat16)], cuda)
    base = [0x00123450, 0x00ABC000]
    vg.set_device_base(base)
    for replay in range(3):
        check_allgather(vg, counts, offs, K.SYMM_AUTO, 0, seed=replay)
        check_reduce_scatter(vg, counts, offs, 0, 10 + replay)
        check_reduce_scatter_bf16(vg, counts, offs, 0, 20 + replay, _weights(n))
        want = vg.dev_base[0] + 1           # the replay's first AG channel launch
        for r in range(n):
            words = vg.signal_words(r, n).cpu().numpy().astype(np.int64)
            assert (words == want).all(), f"rank {r} start-barrier slots {words} != {want}"
        vg.add_device_base(0, 1)           # one AG launch per "replay"
        vg.add_device_base(1, 2)           # two RS launches


def test_missing_rank_times_out_and_is_reported(cuda):
    """Fault injection: rank 0 of a 2-rank all-gather is launched alone (the
    real per-rank entry point, one launch) and rank 1 never joins. Rank 0's
    kernel must give up after the (shortened) spin limit, the sticky status
    must say so, and the asynchronous StatusWatch the step driver uses must
    raise CollectiveFault instead of letting the step train on its output."""
    import ctypes
    vg = VirtualGroup(2, [("unit", 4096, torch.bfloat16)], cuda)
    counts = [2048, 2048]
    src = [torch.randn(2048, device=cuda) for _ in range(2)]
    watch = K.StatusWatch()
    lib = K.load()
    K.set_symm_timeout_ms(200)
    try:
        t0 = time.time()
        K._check(lib.het_symm_allgather_pack(ctypes.byref(vg.desc[0]), src[0].data_ptr(),
                                             vg.offsets["unit"], K._i64(counts),
                                             K._i64([0, 2048]), 1, 0, K.SYMM_PEER, 4,
                                             torch.cuda.current_stream().cuda_stream),
                 "het_symm_allgather_pack")
        watch.record(torch.cuda.current_stream(), "step 7")
        with pytest.raises(K.CollectiveFault, match="step 7"):
            watch.check()
        assert time.time() - t0 < 5.0
        assert K.SymmWorkspace.status(reset=True) == K.HET_SYMM_TIMEOUT
    finally:
        K.set_symm_timeout_ms(10_000)
    # a clean collective afterwards (both ranks, one cooperative launch) reports 0
    vg.epoch[0] = 1
    vg.allgather_pack(src, "unit", 0, counts, [0, 2048])
    watch.record(torch.cuda.current_stream(), "step 8")
    watch.check()
