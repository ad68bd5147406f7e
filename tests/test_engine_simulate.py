"""GPU parity of the plan simulator: gp_simulate (one GPU thread per
seed) against the reference's own simulate() reports (tests/golden/simulate.json, made by
tests/golden/make_golden_simulate.py from oracle/_ref/libref.so), field by field with ==."""
import pytest

from common import golden, problem

pytestmark = pytest.mark.gpu


def test_simulate_vs_reference():
    from paper_2511_00796_b200.engine import Engine
    engines = {}
    cases = golden("simulate.json")
    checked = 0
    for case in cases:
        name = case["config"]
        if name not in engines:
            engines[name] = Engine(problem(name))
        want = case["ref"]
        if "error" in want:
            continue
        reps, used = engines[name].simulate(case["plan"], case["steps"], [case["seed"]], case["sync_every"])
        got = reps[0]
        for k, v in want.items():
            if k == "used_rollout_devices":
                assert used == v, (case["plan_label"], k)
            else:
                assert got[k] == v, (case["plan_label"], case["steps"], case["seed"], k, got[k], v)
        checked += 1
    assert checked >= 30


def test_simulate_many_seeds_at_once():
    """Replica-parallel: 256 seeds in one launch == one launch per seed."""
    from paper_2511_00796_b200.engine import Engine
    case = golden("simulate.json")[2]
    eng = Engine(problem(case["config"]))
    seeds = list(range(1000, 1256))
    many, _ = eng.simulate(case["plan"], 30, seeds)
    for i in (0, 17, 255):
        one, _ = eng.simulate(case["plan"], 30, [seeds[i]])
        assert one[0] == many[i]
