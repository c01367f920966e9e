"""Plan contract (JSON schemas, validation, errors) and the per-rank HBM
layout derived from it. CPU only."""
import json
import re
from pathlib import Path

import pytest

import paper_2411_01075_b200 as H
from paper_2411_01075_b200.configs import build_job
from paper_2411_01075_b200.layout import ALIGN, RankLayout, root_shard_plan
from paper_2411_01075_b200.model import ARCHS

GOLD = Path(__file__).resolve().parent / "golden"
ROOT = Path(__file__).resolve().parent.parent


def test_plan_json_roundtrip_and_unknown_fields(tmp_path):
    job = build_job("bert_large", 4, measured=True)
    p = tmp_path / "plan.json"
    H.save_plan(job.plan, p)
    again = H.load_plan(p)
    assert H.plan_to_dict(again) == H.plan_to_dict(job.plan)
    doc = json.loads(p.read_text())
    doc["surprise"] = 1
    with pytest.raises(H.InputError, match="unknown fields"):
        H.plan_from_dict(doc)
    doc.pop("surprise")
    doc["assignments"][0]["microbatch"] = 1.5
    with pytest.raises(H.InputError, match="integer"):
        H.plan_from_dict(doc)


def test_cluster_and_model_schema_errors():
    with pytest.raises(H.InputError, match="missing"):
        H.cluster_from_dict({"gpus": []})
    with pytest.raises(H.InputError, match="non-empty"):
        H.cluster_from_dict({"gpus": [], "comm": {"allgather_ms": 1, "reducescatter_ms": 1}})
    with pytest.raises(H.InputError, match="unique"):
        H.cluster_from_dict({"gpus": [{"id": "a", "memory_gib": 1, "profile_key": "k"}] * 2,
                             "comm": {"allgather_ms": 1, "reducescatter_ms": 1}})
    with pytest.raises(H.InputError, match=">= 1"):
        H.model_from_dict({"layers": 0, "params_per_layer": 1, "global_batch": 1})
    c = H.cluster_from_dict({"gpus": [{"id": "a", "memory_gib": 1.5, "profile_key": "k"}],
                             "comm": {"allgather_ms": 1, "reducescatter_ms": 2}})
    assert c.gpus[0].memory_capacity == int(round(1.5 * 2 ** 30))
    assert c.mem_cap_fraction == 0.8 and c.comm.uneven_overhead == 0.15
    assert H.cluster_from_dict(H.cluster_to_dict(c)) == c


def test_error_hierarchy():
    assert issubclass(H.InputError, H.HetplanError)
    assert issubclass(H.InfeasibleError, H.HetplanError)
    assert issubclass(H.FitError, H.InputError)
    assert issubclass(H.SizeGuardError, H.InputError)


def test_validator_catches_each_constraint():
    job = build_job("llama_1b3", 4)
    mm = job.perf.memory_models()
    assert H.validate_plan(job.plan, job.cluster, job.model, mm) == []
    d = H.plan_to_dict(job.plan)
    d["assignments"][0]["batch"] += 1
    v = H.validate_plan(H.plan_from_dict(d), job.cluster, job.model, mm)
    assert {x.constraint for x in v} >= {"I"}
    d = H.plan_to_dict(job.plan)
    d["assignments"] = d["assignments"][:-1]
    with pytest.raises(H.InputError):
        H.validate_plan(H.plan_from_dict(d), job.cluster, job.model, mm)


@pytest.mark.parametrize("case", range(0, 150, 7))
def test_rank_layouts_partition_every_unit(case):
    c = json.loads((GOLD / "sharding.json").read_text())["cases"][case]
    n = len(c["ratios"])
    md = H.ModelSpec(c["layers"], c["unit_params"], 1)
    shards = H.assign_unit_shards(c["ratios"], md)
    root = H.assign_unit_shards(c["ratios"], H.ModelSpec(1, 1000 + case, 1))
    lays = [RankLayout.build(shards, root, c["unit_params"], 1000 + case, r) for r in range(n)]
    for u in range(c["layers"] + 1):
        size = c["unit_params"] if u < c["layers"] else 1000 + case
        covered = sorted((lay.offsets[u][r], lay.counts[u][r]) for r, lay in enumerate(lays))
        pos = 0
        for off, cnt in covered:
            assert off == pos
            pos += cnt
        assert pos == size
    for lay in lays:
        assert all(o % ALIGN == 0 for o in lay.local_off)       # 256 B aligned fp32 ranges
        ends = [o + lay.counts[u][lay.rank] for u, o in enumerate(lay.local_off)]
        assert all(e <= nxt for e, nxt in zip(ends, list(lay.local_off[1:]) + [lay.local_len]))
        assert lay.owned_params == sum(cnt[lay.rank] for cnt in lay.counts)


def test_layout_rejects_bad_plans():
    arch = ARCHS["tiny_gpt"]
    job = build_job("tiny_gpt", 2)
    with pytest.raises(H.InputError):
        RankLayout.from_plan(job.plan, arch.unit_params + 1, arch.root_params, 0)
    with pytest.raises(H.InputError):
        RankLayout.from_plan(job.plan, arch.unit_params, arch.root_params, 5)
    rs = root_shard_plan(job.plan, arch.root_params)
    assert sum(rs.shards[0]) == arch.root_params


def test_unit_param_counts_match_survey():
    # U = 12d^2+13d (GPT/BERT), 4d^2+3 d ffn+2d (Llama)
    assert ARCHS["tiny_gpt"].unit_params == 789_760
    assert ARCHS["gpt2_small"].unit_params == 7_087_872
    assert ARCHS["bert_large"].unit_params == 12_596_224
    assert ARCHS["llama_1b3"].unit_params == 51_384_320


def test_header_symbols_are_exported():
    """The C-ABI library loads on a CPU-only host and exports every entry
    point include/hetstep.h declares (no compute calls without a GPU)."""
    import ctypes

    from paper_2411_01075_b200 import _build, hetstep
    lib = ctypes.CDLL(str(_build.build_step()))
    hdr = (ROOT / "include" / "hetstep.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(het_\w+)\(", hdr, re.M))
    assert declared == set(hetstep.EXPORTS)
    for sym in declared:
        assert hasattr(lib, sym), sym
    lib.het_version.restype = ctypes.c_char_p
    assert lib.het_version().decode().startswith("hetstep")


def _relay_link_bytes(counts):
    """Per-rank (egress, ingress) of the relay all-gather as relay_plan() in
    csrc/hetstep_symm.cu schedules it: pair i-th largest A with i-th smallest
    B, A hands f of its range to B only, B forwards it to the other N-2."""
    n = len(counts)
    eg = [(n - 1) * c for c in counts]
    order = sorted(range(n), key=lambda j: -counts[j])
    for i in range(n // 2):
        a, b = order[i], order[n - 1 - i]
        if counts[a] <= counts[b]:
            break
        f = (counts[a] - counts[b]) * (n - 1) / (2.0 * (n - 2) * counts[a])
        eg[a] -= (n - 2) * f * counts[a]
        eg[b] += (n - 2) * f * counts[a]
    total = sum(counts)
    return eg, [total - c for c in counts]


def test_ag_relay_policy_link_model():
    from paper_2411_01075_b200 import hetstep as K
    T = 6 * 10**8
    # 2:1 at N=4: balanced egress 3S/4, bound moves to the small owners' ingress 5S/6
    c = [2 * T, T, 2 * T, T]
    eg, ing = _relay_link_bytes(c)
    S = sum(c)
    assert max(eg) == pytest.approx(0.75 * S)
    assert max(max(eg), max(ing)) == pytest.approx(5 * S / 6)
    assert K.ag_symm_policy(c, 4) == K.SYMM_RELAY
    # no gain: even shards, N=2, geometric (7% model margin), zero-count ranks
    assert K.ag_symm_policy([T] * 4, 4) == K.SYMM_AUTO
    assert K.ag_symm_policy([2 * T, T], 2) == K.SYMM_AUTO
    assert K.ag_symm_policy([T >> i for i in range(4)], 4) == K.SYMM_AUTO
    assert K.ag_symm_policy([T, 0, T, 0], 4) == K.SYMM_AUTO
    assert K.ag_symm_policy([0, 0, 0, 0], 4) == K.SYMM_AUTO
    # the Python model is the kernel's pairing with its 1.25x share: 2:1 lands on
    # the small owners' ingress bound 5S/6
    assert K.relay_link_bytes(c, 4) == pytest.approx(5 * S / 6)
    # without an NVLS multicast object the comparison is against plain push only:
    # geometric and two-owner shapes then take the relay
    assert K.ag_symm_policy([T >> i for i in range(4)], 4, multicast=False) == K.SYMM_RELAY
    assert K.ag_symm_policy([T, 0, T, 0], 4, multicast=False) == K.SYMM_RELAY
    assert K.ag_symm_policy([T] * 4, 4, multicast=False) == K.SYMM_AUTO
    # the relay never raises any rank's egress above the plain push maximum
    for c in ([5, 1, 1, 1], [9, 4, 2, 1], [3, 3, 1, 1, 2, 2, 1, 1], [7, 0, 0, 0]):
        eg, _ = _relay_link_bytes(c)
        assert max(eg) <= (len(c) - 1) * max(c) + 1e-9


def test_helper_plan_balances_links():
    """HET_SYMM_HELPERS plan (csrc/hetstep_symm.cu helper_plan), host-only:
    pieces go from heavy owners to light helpers, never to the owner itself,
    and the plan's largest per-link load is never above the plain peer route's
    and reaches the ingress bound on single-owner units (S at N ranks instead
    of (N-1) S)."""
    from paper_2411_01075_b200 import hetstep as K
    S = 7_087_872
    cases = [[S, 0, 0, 0], [0] * 6 + [S, 0], [0, 0, 0, 0, 1_771_968, 0, 5_315_904, 0],
             [2000, 1000, 2000, 1000], [1000] * 4, [S, 0], [5, 1, 1, 1], [0, 0, 3, 0, 0]]
    for c in cases:
        offs = [sum(c[:j]) for j in range(len(c))]
        for op in (K.OP_AG, K.OP_RS, K.OP_RS_BF16):
            p = K.helper_plan(op, c, offs)
            plain = K.plain_link_bytes(op, c)
            assert max(p["link_bytes"]) <= plain * (1 + 1e-9) + 64, (c, op)
            for o, h in p["pieces"]:
                assert o != h and c[o] > c[h], (c, op, o, h)
            if len(c) >= 3 and sorted(c)[-2] == 0 and sum(c) > 10_000 and op != K.OP_RS_BF16:
                es = 2 if op == K.OP_AG else 4
                assert max(p["link_bytes"]) == pytest.approx(es * sum(c), rel=1e-3), (c, op)
        if len(c) < 3:
            assert K.helper_plan(K.OP_AG, c, offs)["pieces"] == []


@pytest.mark.parametrize("n", [2, 4, 8])
def test_default_route_table_is_all_fused(n, monkeypatch):
    """Round-2 default (hetstep.OWNER_FUSED = "all"): every unit shape of the
    three bench plans routes through the fused kernels for AG and both RS forms,
    so an all-fused step is graph-capturable; OWNER_FUSED = "none" restores the
    NCCL ring for near-single-owner units at N >= 4 only."""
    from paper_2411_01075_b200 import hetstep as K
    from paper_2411_01075_b200.configs import build_job
    from paper_2411_01075_b200.layout import RankLayout
    for name in ("gpt2_small", "bert_large", "llama_1b3"):
        job = build_job(name, n, measured=True)
        lay = RankLayout.from_plan(job.plan, job.arch.unit_params, job.arch.root_params, 0)
        for c in lay.counts:
            for op in ("ag", "rs", "rs16"):
                assert K.route_collective(op, c, n, True) == "symm", (name, n, op, c)
                assert K.route_collective(op, c, n, False) == "nccl"
        monkeypatch.setattr(K, "OWNER_FUSED", "none")
        for c in lay.counts:
            owner_like = n >= 4 and max(c) >= 0.75 * sum(c)
            want = "nccl" if owner_like else "symm"
            assert K.route_collective("ag", c, n, True) == want, (name, n, c)
            assert K.route_collective("rs16", c, n, True) == want, (name, n, c)
        monkeypatch.setattr(K, "OWNER_FUSED", "all")


def test_device_epoch_bookkeeping(monkeypatch):
    """SymmWorkspace device-epoch mode (the multi-rank CUDA graph), host side:
    inside a capture each launch passes EPOCH_DEVICE | its offset from the
    capture start, end_device_epochs queues one base advance per channel by the
    step's launch count, restores the host counters (the capture ran nothing)
    and returns those deltas; advance_host after each replay keeps the host
    counters equal to the device bases."""
    from paper_2411_01075_b200 import hetstep as K
    calls = []

    class Lib:
        def het_symm_epoch_set(self, desc, ch, v, st):
            calls.append(("set", ch, v))
            return 0

        def het_symm_epoch_add(self, desc, ch, d, st):
            calls.append(("add", ch, d))
            return 0

    monkeypatch.setattr(K, "load", lambda: Lib())
    monkeypatch.setattr(K, "_stream", lambda st: 0)      # no CUDA here
    ws = K.SymmWorkspace.__new__(K.SymmWorkspace)
    ws.desc, ws.epoch, ws._dev_epoch0 = K.HetSymm(), [7, 11], None
    assert ws._next_epoch(0) == 8                      # host epochs
    ws.begin_device_epochs(None)
    assert calls == [("set", 0, 8), ("set", 1, 11)]
    got = [ws._next_epoch(0), ws._next_epoch(1), ws._next_epoch(1), ws._next_epoch(0)]
    assert got == [K.EPOCH_DEVICE | 1, K.EPOCH_DEVICE | 1, K.EPOCH_DEVICE | 2,
                   K.EPOCH_DEVICE | 2]
    deltas = ws.end_device_epochs(None)
    assert deltas == [2, 2] and calls[-2:] == [("add", 0, 2), ("add", 1, 2)]
    assert ws.epoch == [8, 11] and ws._dev_epoch0 is None
    for _ in range(3):                                 # three replays
        ws.advance_host(deltas)
    assert ws.epoch == [14, 17]
    assert ws._next_epoch(1) == 18                     # an eager call continues the sequence
    with pytest.raises(K.InputError):
        ws.end_device_epochs(None)
