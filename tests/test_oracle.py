"""CPU: pins the C restatement (oracle/) to the reference's golden vectors."""
import json

import pytest

from common import CONFIGS, golden, problem
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
