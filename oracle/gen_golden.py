#!/usr/bin/env python
"""Generate tests/golden/*.json by running the REFERENCE implementation
(`hetplan`, imported read-only from /root/reference/pkg/src) — TEST
INFRASTRUCTURE ONLY; run in the build container, never on the GPU box:

  python oracle/gen_golden.py [--reference /root/reference/pkg/src]

Every file stores the inputs (reference-schema documents) next to the
reference's outputs, so the CPU test-suite can pin this repo's planner,
sharding, fits, validator and Eq. 1 weighting without the reference present.
Instance generators mirror the reference's own test generators
(pkg/tests/conftest.py:22-157: affine profiles with jitter, ample/scarce
memory, 30% idle permission) and add the B200 benchmark configurations.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "tests" / "golden"


def affine_doc(key, fwd_slope, fwd_icept=0.0, mem0=2.0, mem_slope=0.25, max_m=8, bwd_factor=2.0,
               jitter=None, rng=None):
    def noisy(v):
        return v if jitter is None else v * (1.0 + jitter * rng.uniform(-1.0, 1.0))
    return {"profile_key": key,
            "fwd_ms": [[m, noisy(fwd_icept + fwd_slope * m)] for m in range(1, max_m + 1)],
            "bwd_ms": [[m, noisy(bwd_factor * (fwd_icept + fwd_slope * m))]
                       for m in range(1, max_m + 1)],
            "compute_mem_gib": [[m, mem0 + mem_slope * m] for m in range(1, max_m + 1)]}


def random_instance(rng, R):
    """Same distribution as the reference's conftest.random_instance."""
    while True:
        n = int(rng.integers(1, 5))
        batch = int(rng.integers(2, 13))
        mem_slope = 0.2 + 0.3 * rng.random()
        docs, caps = [], []
        for i in range(n):
            max_m = int(rng.integers(2, 13))
            docs.append(affine_doc(f"g{i}", fwd_slope=0.5 + 4.0 * rng.random(),
                                   fwd_icept=2.0 * rng.random(), mem0=1.0 + 3.0 * rng.random(),
                                   mem_slope=mem_slope, max_m=max_m,
                                   bwd_factor=1.0 + 2.0 * rng.random(), jitter=0.15, rng=rng))
            mem0 = docs[-1]["compute_mem_gib"][0][1] - mem_slope
            if rng.random() < 0.5:
                caps.append(mem0 + mem_slope * batch + 8.0)
            else:
                caps.append(mem0 + mem_slope * float(rng.integers(0, batch + 1)))
        try:
            perf_of(R, docs)
        except R.FitError:
            continue
        cluster = {"gpus": [{"id": f"{d['profile_key']}-{i}", "memory_gib": c,
                             "profile_key": d["profile_key"]}
                            for i, (c, d) in enumerate(zip(caps, docs))],
                   "comm": {"allgather_ms": float(rng.choice([0.05, 1.0, 25.0])),
                            "reducescatter_ms": float(rng.choice([0.05, 1.0, 25.0])),
                            "uneven_overhead": 0.15},
                   "mem_cap_fraction": 1.0}
        model = {"layers": int(rng.integers(1, 7)),
                 "params_per_layer": int(rng.integers(100_000, 5_000_000)),
                 "global_batch": batch, "bytes_per_param_state": 16}
        return {"profiles": docs, "cluster": cluster, "model": model,
                "allow_idle": bool(rng.random() < 0.3)}


def perf_of(R, docs):
    models = {}
    for d in docs:
        c, m = R.profile_from_dict(d)
        models[c.profile_key] = R.fit_perf_model(c, m)
    return R.ClusterPerf(models)


def run_planner(R, inst, brute=False):
    perf = perf_of(R, inst["profiles"])
    cl = R.cluster_from_dict(inst["cluster"])
    md = R.model_from_dict(inst["model"])
    try:
        if brute:
            return {"plan": R.plan_to_dict(R.brute_force_optimize(
                cl, md, perf, allow_idle=inst["allow_idle"]))}
        res = R.dp_optimize_detailed(cl, md, perf, allow_idle=inst["allow_idle"])
        rep = res.report.to_dict()
        for k in ("wall_time_s", "threads"):
            rep.pop(k)
        return {"plan": R.plan_to_dict(res.plan), "report": rep}
    except R.HetplanError as e:
        return {"error": type(e).__name__, "message": str(e)}


def dump(name, doc):
    OUT.mkdir(parents=True, exist_ok=True)
    (OUT / name).write_text(json.dumps(doc, sort_keys=True, separators=(",", ":")) + "\n")
    print(f"wrote {name} ({(OUT / name).stat().st_size / 1024:.0f} KiB)")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--reference", default="/root/reference/pkg/src")
    ap.add_argument("--instances", type=int, default=300)
    ap.add_argument("--skip-64", action="store_true")
    args = ap.parse_args()
    sys.path.insert(0, args.reference)
    sys.path.insert(0, str(ROOT))
    import hetplan as R
    from importlib import resources
    meta = {"reference": "hetplan " + R.__version__, "numpy": np.__version__,
            "generated": time.strftime("%Y-%m-%d"), "script": "oracle/gen_golden.py"}

    # 1. random planner instances (DP report + brute-force oracle)
    rng = np.random.default_rng(2024)
    cases = []
    for _ in range(args.instances):
        inst = random_instance(rng, R)
        inst["dp"] = run_planner(R, inst)
        inst["bf"] = run_planner(R, inst, brute=True)
        cases.append(inst)
    dump("planner_random.json", {"meta": meta, "cases": cases})

    # 2. the paper-era fixtures shipped with the reference (data, not code)
    fx = lambda n: json.loads(resources.files("hetplan").joinpath("fixtures")  # noqa: E731
                              .joinpath(n).read_text())
    fixture_cases = []
    combos = [("cluster_mixed_8gpu.json", "profiles_mixed_8gpu.json",
               ["model_bert_large.json", "model_bert_xlarge.json", "model_gpt_2_7b.json",
                "model_tiny_llama.json", "model_llama_3b.json", "model_vit_g.json"])]
    if not args.skip_64:
        combos.append(("cluster_mixed_64gpu.json", "profiles_mixed_64gpu.json",
                       ["model_gpt_6_7b.json"]))
    for cname, pname, models in combos:
        for mname in models:
            inst = {"name": f"{cname}+{mname}", "profiles": fx(pname), "cluster": fx(cname),
                    "model": fx(mname), "allow_idle": False}
            t0 = time.time()
            inst["dp"] = run_planner(R, inst)
            inst["reference_seconds"] = time.time() - t0
            fixture_cases.append(inst)
    dump("planner_fixtures.json", {"meta": meta, "cases": fixture_cases})

    # 3. the B200 benchmark configurations (emulated tiers) at 1/2/4/8 GPUs
    from paper_2411_01075_b200.configs import CONFIGS, cluster_doc, tier_profile
    from paper_2411_01075_b200.model import ARCHS
    bcases = []
    for name, cfg in sorted(CONFIGS.items()):
        arch = ARCHS[cfg.arch]
        for n in (1, 2, 4, 8):
            tiers = list(cfg.tiers[:n])
            inst = {"name": f"{name}@{n}",
                    "profiles": [tier_profile(arch, t) for t in sorted(set(tiers))],
                    "cluster": cluster_doc(arch, tiers),
                    "model": {"layers": arch.layers, "params_per_layer": arch.unit_params,
                              "global_batch": cfg.batch_per_gpu * n},
                    "allow_idle": False}
            inst["dp"] = run_planner(R, inst)
            bcases.append(inst)
    dump("planner_b200_configs.json", {"meta": meta, "cases": bcases})

    # 4. unit shards: reference test vectors, planner-style quanta, real model sizes
    shard_cases = [([0.75, 0.25], 2, 1000), ([0.25] * 4, 4, 1200), ([1.0, 0.0], 3, 999),
                   ([1 / 3 + 1e-12, 1 / 3, 1 / 3 - 1e-12], 6, 9000), ([0.5, 0.3, 0.2], 5, 977),
                   ([0.6, 0.4], 2, 10), ([683 / 1024, 341 / 1024], 12, 7_087_872),
                   ([1.0], 24, 12_596_224), ([368 / 1024, 656 / 1024], 4, 789_760)]
    srng = np.random.default_rng(7)
    for _ in range(150):
        n = int(srng.integers(1, 9))
        q = srng.multinomial(1024, srng.dirichlet(np.ones(n) * float(srng.choice([0.2, 1, 5]))))
        ratios = [int(x) / 1024 for x in q]
        L = int(srng.integers(1, 40))
        U = int(srng.choice([int(srng.integers(1, 5000)), int(srng.integers(10**5, 6 * 10**7))]))
        shard_cases.append((ratios, L, U))
    srecs = []
    for ratios, L, U in shard_cases:
        md = R.model_from_dict({"layers": L, "params_per_layer": U, "global_batch": 1})
        sp = R.assign_unit_shards(ratios, md)
        srecs.append({"ratios": ratios, "layers": L, "unit_params": U,
                      "shards": [list(v) for v in sp.shards],
                      "offsets": [list(v) for v in sp.offsets], "uneven_units": sp.uneven_units})
    dump("sharding.json", {"meta": meta, "cases": srecs})

    # 5. Eq. 1: reference weighted_combine on random fixtures
    grng = np.random.default_rng(0)
    wrecs = []
    for _ in range(60):
        f = R.random_fixture(grng)
        means = [g.mean(axis=0) for g in f.sample_grads]
        wrecs.append({"means": [m.tolist() for m in means], "batches": list(f.batches),
                      "weighted": R.weighted_combine(means, f.batches).tolist(),
                      "full_batch_mean": R.full_batch_mean(f.sample_grads).tolist()})
    rep = R.run_check(fixtures=200, seed=0)
    dump("weighted_combine.json", {"meta": meta, "cases": wrecs,
                                   "run_check_200_seed0": {
                                       "max_rel_error": rep.max_rel_error,
                                       "max_unweighted_rel_error": rep.max_unweighted_rel_error}})

    # 6. fitted perf models (lstsq) for every profile document used above
    docs = {}
    for inst in cases[:40] + fixture_cases + bcases:
        for d in inst["profiles"]:
            docs[json.dumps(d, sort_keys=True)] = d
    frecs = []
    for d in docs.values():
        try:
            frecs.append({"profile": d, "perf": R.perf.perf_to_dict(perf_of(R, [d]))})
        except R.FitError as e:
            frecs.append({"profile": d, "error": str(e)})
    dump("perf_fits.json", {"meta": meta, "cases": frecs})

    # 7. validator verdicts on produced and damaged plans
    vrecs = []
    for inst in fixture_cases[:3] + bcases[:8]:
        if "plan" not in inst["dp"]:
            continue
        for mutate in ("none", "batch", "ratio", "iteration", "state_mem"):
            plan = json.loads(json.dumps(inst["dp"]["plan"]))
            a0 = plan["assignments"][0]
            if mutate == "batch":
                a0["batch"] += 1
            elif mutate == "ratio":
                a0["state_ratio"] = min(1.0, a0["state_ratio"] + 0.01)
            elif mutate == "iteration":
                plan["predicted_iteration_ms"] *= 1.01
            elif mutate == "state_mem":
                a0["predicted_state_mem_gib"] += 1.0
            perf = perf_of(R, inst["profiles"])
            v = R.validate_plan(R.plan_from_dict(plan), R.cluster_from_dict(inst["cluster"]),
                                R.model_from_dict(inst["model"]), perf.memory_models())
            vrecs.append({"instance": inst.get("name"), "mutation": mutate, "plan": plan,
                          "profiles": inst["profiles"], "cluster": inst["cluster"],
                          "model": inst["model"],
                          "violations": [[x.constraint, x.gpu_id] for x in v]})
    dump("validate.json", {"meta": meta, "cases": vrecs})


if __name__ == "__main__":
    main()
