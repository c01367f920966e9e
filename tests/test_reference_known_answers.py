"""The reference's own known-answer tests, restated against this package's
drop-in API (reference pkg/tests/test_sharding.py,
test_planner.py, test_acceptance.py, test_gradcheck.py)."""
import pytest

import paper_2411_01075_b200 as H

GIB = 2 ** 30


def affine(key, slope, icept=0.0, mem0=2.0, mslope=0.25, max_m=8, bwd=2.0):
    return {"profile_key": key,
            "fwd_ms": [[m, icept + slope * m] for m in range(1, max_m + 1)],
            "bwd_ms": [[m, bwd * (icept + slope * m)] for m in range(1, max_m + 1)],
            "compute_mem_gib": [[m, mem0 + mslope * m] for m in range(1, max_m + 1)]}


def perf(docs):
    out = {}
    for d in docs:
        c, m = H.profile_from_dict(d)
        out[c.profile_key] = H.fit_perf_model(c, m)
    return H.ClusterPerf(out)


def cluster(caps, keys, ag=1.0, rs=1.0, frac=1.0):
    return H.cluster_from_dict({"gpus": [{"id": f"{k}-{i}", "memory_gib": c, "profile_key": k}
                                         for i, (c, k) in enumerate(zip(caps, keys))],
                                "comm": {"allgather_ms": ag, "reducescatter_ms": rs},
                                "mem_cap_fraction": frac})


def slope_instance(slopes, batch, layers=1, ag=0.001, rs=0.001):
    docs = [affine(f"g{i}", s, mem0=1.0, max_m=batch) for i, s in enumerate(slopes)]
    return (cluster([64.0] * len(slopes), [d["profile_key"] for d in docs], ag, rs),
            H.ModelSpec(layers, 1000, batch), perf(docs))


def test_three_to_one_ratio_over_two_units():          # test_sharding.py:9-15
    p = H.assign_unit_shards([0.75, 0.25], H.ModelSpec(2, 1000, 1))
    assert p.shards == ((500, 500), (1000, 0))
    assert p.offsets == ((0, 500), (0, 1000))
    assert p.uneven_units == 1


def test_even_and_single_owner_shards():                # test_sharding.py:18-42
    assert all(v == (300,) * 4 for v in
               H.assign_unit_shards([0.25] * 4, H.ModelSpec(4, 1200, 1)).shards)
    p = H.assign_unit_shards([1.0, 0.0], H.ModelSpec(3, 999, 1))
    assert p.uneven_units == 3 and all(v == (999, 0) for v in p.shards)
    assert H.assign_unit_shards([1 / 3 + 1e-12, 1 / 3, 1 / 3 - 1e-12],
                                H.ModelSpec(6, 9000, 1)).uneven_units == 0
    with pytest.raises(H.InputError, match="sum"):
        H.assign_unit_shards([0.5, 0.4], H.ModelSpec(1, 10, 1))


def test_known_optimum_three_speed_cluster():           # test_planner.py:35-44
    c, m, p = slope_instance([1.0, 2.0, 4.0], batch=14)
    plan = H.dp_optimize(c, m, p)
    assert tuple(a.batch for a in plan.assignments) == (8, 4, 2)
    assert plan.predicted_layer_fwd_ms == pytest.approx(8.0, rel=1e-12)
    assert plan.predicted_layer_bwd_ms == pytest.approx(24.0, rel=1e-12)
    assert plan.predicted_iteration_ms == pytest.approx(32.0, rel=1e-12)


def test_per_gpu_layer_latency_formula():               # test_planner.py:62-71
    c, m, p = slope_instance([2.0], batch=8, ag=5.0, rs=7.0)
    lat = H.per_gpu_layer_latency(c.gpus[0], p, c.comm, 2, 2, 0.0)
    assert (lat.t_fwd_ms, lat.t_bwd_ms) == pytest.approx((8.0, 24.0))
    lat = H.per_gpu_layer_latency(c.gpus[0], p, c.comm, 1, 1, 0.0)
    assert (lat.t_fwd_ms, lat.t_bwd_ms) == pytest.approx((5.0, 12.0))


def test_complexity_budget_and_tie_break():             # test_planner.py:74-79, 163-169
    assert H.complexity_budget(1, 1) == 1
    assert H.complexity_budget(2, 4) == 86
    c, m, p = slope_instance([1.0], batch=6)
    a = H.dp_optimize(c, m, p).assignments[0]
    assert (a.microbatch, a.num_microbatches) == (1, 6)


def test_state_water_fill_853_171():                    # test_planner.py:221-239
    docs = [affine("k", 1.0, mem0=5.0, mslope=1.0, max_m=4)]
    c = cluster([24.0, 12.0], ["k", "k"], 0.01, 0.01)
    m = H.ModelSpec(2, (12 * GIB) // (16 * 2), 2)
    plan = H.dp_optimize(c, m, perf(docs))
    assert [a.state_ratio for a in plan.assignments] == [853 / 1024, 171 / 1024]


def test_memory_cap_forces_layered_accumulation():      # test_acceptance.py:157-168
    docs = [affine(f"g{i}", 1.0, icept=1.0, mem0=4.0, mslope=1.0) for i in range(2)]
    c = cluster([6.5, 6.5], ["g0", "g1"], 0.05, 0.05)
    plan = H.dp_optimize(c, H.ModelSpec(6, 1000, 16), perf(docs))
    assert {(a.microbatch, a.num_microbatches) for a in plan.assignments} == {(2, 4)}


def test_infeasibility_classes():                       # test_planner.py:103-127
    c, m, p = slope_instance([1.0, 1.0, 1.0], batch=2)
    with pytest.raises(H.InfeasibleError, match="constraint I"):
        H.dp_optimize(c, m, p)
    assert sum(a.idle for a in H.dp_optimize(c, m, p, allow_idle=True).assignments) == 1
    docs = [affine("k", 1.0, mem0=2.0, mslope=0.25, max_m=4)]
    with pytest.raises(H.InfeasibleError, match="constraint III"):
        H.dp_optimize(cluster([3.0, 3.0], ["k", "k"], 0.01, 0.01),
                      H.ModelSpec(2, 2 * GIB // 16, 4), perf(docs))
    with pytest.raises(H.SizeGuardError):
        c6, m6, p6 = slope_instance([1.0] * 6, batch=6)
        H.brute_force_optimize(c6, m6, p6)


def test_eq1_reweighting_1000_fixtures():               # test_acceptance.py:93-100
    rep = H.run_check(fixtures=1000, seed=0, tolerance=1e-12)
    assert rep.passed and rep.max_rel_error <= 1e-12
    assert rep.max_unweighted_rel_error > rep.max_rel_error


def test_partition_state_rederives():                   # test_planner.py:242-251
    c, m, p = slope_instance([1.0, 2.0], batch=8)
    plan = H.dp_optimize(c, m, p)
    again = H.partition_state(plan, c, m)
    assert [a.state_ratio for a in again.assignments] == [a.state_ratio for a in plan.assignments]
    assert again.unit_shards == plan.unit_shards
