"""CPU: pins the C restatement (oracle/) to the reference's golden vectors."""
import json

import pytest

from common import CONFIGS, golden, problem, random_train_sets
from oracles import Oracle


def _strip(plan):
    plan = dict(plan)
    for k in ("format", "cluster_fingerprint", "calibration_fingerprint", "workload_fingerprint"):
        plan.pop(k, None)
    return plan


def test_desk_plan_golden():
    """proj/out/desk/plan.json: the committed reference output."""
    out = Oracle(problem("c1_desk_mixed")).schedule(eta=-1)
    out.pop("trace")
    out.pop("evaluated_partitions")
    assert out == _strip(golden("desk_plan.json"))


@pytest.mark.parametrize("key", sorted(golden("schedules.json")))
def test_schedule_matches_reference(key):
    g = golden("schedules.json")[key]
    name, eta = key.split("/eta=")
    out = Oracle(problem(name)).schedule(eta=int(eta))
    trace = out.pop("trace")
    out.pop("evaluated_partitions")
    assert out == _strip(g["plan"])
    assert trace == g["trace"]


@pytest.mark.parametrize("name", CONFIGS)
def test_constrained_search_matches_reference(name):
    orc = Oracle(problem(name))
    for case in golden("train_search.json")[name]:
        got = orc.constrained_search(case["ids"], case["window"])
        ref = case["ref"]
        assert got["found"] == ref["found"]
        assert got["layouts"] == case["layouts"]
        if ref["found"]:
            assert got["cost"] == ref["cost"]  # bit-exact
            assert got["stages"] == ref["stages"]


def test_enumeration_order_and_counts():
    """Layout rank == position in enumerate_train_candidates' distinct block lists."""
    orc = Oracle(problem("c2_16gpu"))
    for ids_key, g in golden("train_candidates.json").items():
        ids = json.loads(ids_key)
        assert orc.train_space(ids) == len(g["block_lists"])
        got = orc.constrained_search(ids, 3)
        # exhaustive argmin over the product space (tests/test_train_search.cpp:26-54)
        best = None
        for c in g["candidates"]:
            if c["fits"] and (best is None or c["cost"] < best["cost"]):
                best = c
        assert got["found"] == (best is not None)
        if best:
            assert got["cost"] == best["cost"]
            blocks = [s["devices"] for s in got["stages"]]
            assert g["block_lists"].index(blocks) == got["rank"]


def test_ranges_partition_the_space():
    orc = Oracle(problem("c3_64gpu"))
    ids = list(range(0, 64, 3))
    total = orc.train_space(ids)
    full = orc.constrained_search(ids, 2)
    cuts = [0, total // 5, total // 2, total - 3, total]
    parts = [orc.constrained_search(ids, 2, lo=a, hi=b) for a, b in zip(cuts, cuts[1:])]
    assert sum(p["feasible"] for p in parts) == full["feasible"]
    win = min((p for p in parts if p["found"]), key=lambda p: (p["cost"], p["rank"]))
    assert (win["cost"], win["rank"], win["stages"]) == (full["cost"], full["rank"], full["stages"])


@pytest.mark.parametrize("name", CONFIGS)
def test_rollout_side_matches_reference(name):
    """enumerate_configs / solve_milp / weight_sync_cost restated in C == reference."""
    from oracles import config_dict, oracle_configs, oracle_milp, oracle_weight_sync
    p = problem(name)
    orc = Oracle(p)
    T = len(p.cluster.type_names)
    for case in golden("rollout.json")[name]:
        cfgs = oracle_configs(orc, case["rollout"])
        got = [config_dict(c, T) for c in cfgs]
        want = [{k: c[k] for k in ("type_counts", "tp_per_stage", "throughput")} for c in case["configs"]]
        assert got == want
        B = float(p.workload.batch_rollouts * case["window"])
        rc, res, ents = oracle_milp(orc, cfgs, case["capacities"], B, p.workload.mean_len)
        if "milp_error" in case:
            assert rc != 0
            continue
        m = case["milp"]
        assert rc == 0
        assert res.makespan == m["makespan"]
        assert [(e.replicas, e.workload) for e in ents] == [(e["replicas"], e["workload"]) for e in m["entries"]]
        assert [config_dict(cfgs[e.config], T) for e in ents] == \
            [{k: e[k] for k in ("type_counts", "tp_per_stage", "throughput")} for e in m["entries"]]
        et = [next(t for t, v in enumerate(e["type_counts"]) if v > 0) for e in m["entries"]]
        er = [e["replicas"] for e in m["entries"]]
        assert oracle_weight_sync(orc, case["train"], case["rollout"], et, er, case["window"]) == case["weight_sync"]


@pytest.mark.parametrize("name", CONFIGS + ["t10_tiny", "t8_tiny"])
def test_partition_matches_reference(name):
    from oracles import RefError, oracle_partitions
    orc = Oracle(problem(name))
    for case in golden("partition.json")[name]:
        kw = dict(k=8, seed=case.get("seed", 4276115), force_local=case.get("force_local", False),
                  machine=case["machine"])
        if "error" in case:
            with pytest.raises(RefError):
                oracle_partitions(orc, case["gamma_l"], case["gamma_h"], **kw)
            continue
        got = oracle_partitions(orc, case["gamma_l"], case["gamma_h"], **kw)
        want = [(c["train"], c["objective"], c["compute_fraction"]) for c in case["candidates"]]
        assert got == want, (case["gamma_l"], case["gamma_h"], case["machine"])


def test_table_oracle_vs_reference_goldens():
    """or_constrained_search_tab (the memoised restatement behind train_full.json) reproduces
    every reference constrained_search golden and the plain restatement's winner rank."""
    for name in CONFIGS:
        orc = Oracle(problem(name))
        for case in golden("train_search.json")[name]:
            r = orc.constrained_search_tab(case["ids"], [case["window"]], threads=4)
            cost, rank = r["windows"][case["window"]]
            assert r["layouts"] == case["layouts"]
            if case["ref"]["found"]:
                assert cost == case["ref"]["cost"]
                if case["layouts"] <= 20_000:  # (the plain restatement is slow on big sets)
                    assert rank == orc.constrained_search(case["ids"], case["window"])["rank"]
            else:
                assert rank == -1


def test_table_oracle_per_layout_equals_plain():
    """Per-layout per_step of the memoised restatement == the plain restatement, bitwise,
    on slices of C3/C4/C5 train sets (incl. the 2.42e9-layout C5 bench set)."""
    import numpy as np
    for name in ("c3_64gpu", "c4_256gpu", "c5_1024gpu"):
        p = problem(name)
        orc = Oracle(p)
        for ids in random_train_sets(p.cluster.n, 2, seed=5) + [list(range(p.cluster.n - 1))]:
            total = orc.train_space(ids)
            rs = [(lo, min(total, lo + 1500)) for lo in sorted({0, total // 3, max(0, total - 1500)})]
            tab = orc.layout_costs_tab(ids, rs)
            plain = np.concatenate([orc.layout_costs(ids, a, b) for a, b in rs])
            np.testing.assert_array_equal(tab.view(np.int64), plain.view(np.int64))


def test_full_golden_c4_recomputed():
    """tests/golden/train_full.json's C4 entries recompute identically (the C5 entries take
    minutes of host time and are recomputed by tests/golden/make_golden_full.py)."""
    orc = Oracle(problem("c4_256gpu"))
    for case in golden("train_full.json")["c4_256gpu"]:
        r = orc.constrained_search_tab(case["ids"], list(range(1, 9)))
        assert r["feasible"] == case["feasible"] and r["layouts"] == case["layouts"]
        for w, (c, k) in r["windows"].items():
            assert case["windows"][str(w)] == {"cost": c, "rank": k}


def test_c4_schedule_restatement_equals_reference():
    """The C restatement's whole C4 schedule fixture (schedule_c4_oracle.json) == the unmodified
    reference's own C4 schedule (schedule_c4_reference.json): plan and trace."""
    from common import golden
    r = golden("schedule_c4_reference.json")["c4_256gpu/eta=2"]
    o = golden("schedule_c4_oracle.json")["c4_256gpu/eta=2"]
    assert {k: v for k, v in o.items() if k not in ("trace", "evaluated_partitions", "oracle_seconds")} == r["plan"]
    assert o["trace"] == r["trace"]
