"""GPU: the native batched Algorithm-1 driver (gp_schedule) reproduces the reference's
golden plans + traces exactly, and agrees with the drop-in path at C4 scale."""
import pytest

from common import golden, problem

pytestmark = pytest.mark.gpu


def _strip(plan):
    plan = dict(plan)
    for k in ("format", "cluster_fingerprint", "calibration_fingerprint", "workload_fingerprint"):
        plan.pop(k, None)
    return plan


@pytest.mark.parametrize("key", sorted(golden("schedules.json")))
def test_native_schedule_matches_golden(key):
    from paper_2511_00796_b200.engine import Engine
    name, eta = key.split("/eta=")
    g = golden("schedules.json")[key]
    with Engine(problem(name)) as eng:
        plan, trace = eng.schedule(eta=int(eta), seed=4276115)
    assert plan == _strip(g["plan"])
    assert trace == g["trace"]


def test_native_schedule_desk_golden():
    from paper_2511_00796_b200.engine import Engine
    with Engine(problem("c1_desk_mixed")) as eng:
        plan, _ = eng.schedule(eta=-1, seed=4276115)
    assert plan == _strip(golden("desk_plan.json"))
