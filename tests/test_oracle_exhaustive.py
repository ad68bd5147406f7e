"""The C restatement of the exhaustive rows against the reference's
own outputs (tests/golden/exhaustive.json, made by tests/golden/make_golden_exhaustive.py):
exhaustive_schedule_optimum, the product-space training argmin and brute_milp_unbounded."""
import pytest

from common import golden, problem
from oracles import Oracle, oracle_configs


@pytest.fixture(scope="module")
def gold():
    return golden("exhaustive.json")


def test_exhaustive_optimum(gold):
    for key, want in gold["exhaustive"].items():
        name, window = key.split("/window=")
        got = Oracle(problem(name)).exhaustive(int(window))
        assert got["feasible"] == want["feasible"], key
        assert got["objective"] == want["objective"], key
        assert got["train_set"] == want["train_set"], key


@pytest.mark.parametrize("name", ["t8_tiny", "t10_tiny", "c1_desk_mixed", "c2_16gpu"])
def test_product_space_argmin(gold, name):
    orc = Oracle(problem(name))
    for case in gold["train_candidates"][name]:
        got = orc.train_candidates_search(case["ids"], case["window"])
        assert got["layouts"] == case["candidates"], case["ids"]
        best = case["best"]
        assert got["found"] == (best is not None), case["ids"]
        if best:
            assert got["cost"] == best["cost"], case["ids"]
            assert got["rank"] == best["rank"], case["ids"]
            assert got["stages"] == best["stages"], case["ids"]


@pytest.mark.parametrize("name", ["t8_tiny", "t10_tiny", "c1_desk_mixed", "c2_16gpu"])
def test_brute_milp(gold, name):
    p = problem(name)
    orc = Oracle(p)
    for case in gold["brute_milp"][name]:
        cfgs = oracle_configs(orc, case["ids"])
        assert len(cfgs) == len(case["configs"])
        B = float(p.workload.batch_rollouts * case["window"])
        got = orc.brute_milp(cfgs, case["capacities"], B, p.workload.mean_len)
        want = case["ref"]
        assert got["feasible"] == want["feasible"], case["ids"]
        assert got["theta"] == want["theta"], case["ids"]
        assert got["replica_counts"] == want["replica_counts"], case["ids"]
