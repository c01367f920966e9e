#!/usr/bin/env python
"""Pin the plans `bench.py` actually runs — TEST INFRASTRUCTURE ONLY; run in
the build container (it imports the REFERENCE planner read-only from
/root/reference/pkg/src), never on the GPU box:

  python oracle/gen_golden_bench_plans.py [--reference /root/reference/pkg/src]

For every benchmark configuration (paper_2411_01075_b200/configs.py) at
N = 1, 2, 4, 8 it builds the same cluster JSON (tier HBM budgets, including
per-config overrides) and the same B200-measured tier profiles
(paper_2411_01075_b200/profiles_b200/*.json, the planner input the bench
uses; the analytic tier model where a measured table has no linear tail, as
configs.build_job does) and runs the reference `dp_optimize_detailed` (planner.py:479-643) and
`assign_unit_shards` (sharding.py:48-98) on them. tests/test_golden_planner.py
compares this repo's planner against the stored outputs with ==.
"""
from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(Path(__file__).resolve().parent))

from gen_golden import dump, run_planner  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--reference", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.path.insert(0, args.reference)
    sys.path.insert(0, str(ROOT))
    import hetplan as R
    import numpy as np
    from paper_2411_01075_b200.configs import (CONFIGS, cluster_doc, measured_profiles,
                                               planner_model, tier_profile)
    from paper_2411_01075_b200.model import ARCHS
    meta = {"reference": "hetplan " + R.__version__, "numpy": np.__version__,
            "generated": time.strftime("%Y-%m-%d"), "script": "oracle/gen_golden_bench_plans.py"}
    cases = []
    for name, cfg in sorted(CONFIGS.items()):
        arch = ARCHS[cfg.arch]
        meas = measured_profiles(name)
        if not meas:
            continue
        for n in (1, 2, 4, 8):
            tiers = list(cfg.tiers[:n])
            docs = [meas[t] for t in sorted(set(tiers))]
            try:
                for d in docs:
                    R.fit_perf_model(*R.profile_from_dict(d))
            except R.FitError:   # launch-bound tables: build_job keeps the analytic model
                docs = [tier_profile(arch, t) for t in sorted(set(tiers))]
            inst = {"name": f"{name}@{n}",
                    "profiles": docs,
                    "cluster": cluster_doc(arch, tiers, memory_gib=dict(cfg.memory_gib)),
                    "model": planner_model(arch, cfg.batch_per_gpu * n),
                    "allow_idle": False}
            inst["dp"] = run_planner(R, inst)
            if "plan" in inst["dp"]:
                # the flat layout shards the real units (U params), with the plan's ratios
                sp = R.assign_unit_shards(
                    [a["state_ratio"] for a in inst["dp"]["plan"]["assignments"]],
                    R.model_from_dict({"layers": arch.layers,
                                       "params_per_layer": arch.unit_params,
                                       "global_batch": cfg.batch_per_gpu * n}))
                inst["shards"] = {"shards": [list(v) for v in sp.shards],
                                  "offsets": [list(v) for v in sp.offsets],
                                  "uneven_units": sp.uneven_units}
            cases.append(inst)
    dump("planner_bench_plans.json", {"meta": meta, "cases": cases})


if __name__ == "__main__":
    main()
