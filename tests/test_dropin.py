"""The drop-in proof: the unmodified reference scheduler (oracle/_ref/libref.so) with
libgplan_shim.so interposed reproduces the reference's golden plans exactly, with
every seam call served by the B200 engine."""
import json
import os
import subprocess
import sys

import pytest

from common import ROOT, golden

pytestmark = pytest.mark.gpu
SHIM = os.path.join(ROOT, "paper_2511_00796_b200", "libgplan_shim.so")
REF = os.path.join(ROOT, "oracle", "_ref", "libref.so")


@pytest.mark.skipif(not (os.path.exists(SHIM) and os.path.exists(REF)),
                    reason="libgplan_shim.so / libref.so not built (need /root/reference at build time)")
def test_reference_scheduler_on_engine_matches_golden():
    keys = sorted(golden("schedules.json"))
    env = dict(os.environ, LD_PRELOAD=SHIM)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "dropin_driver.py"), *keys],
                       capture_output=True, text=True, env=env, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == len(keys)
    for line in lines:
        g = golden("schedules.json")[line["key"]]
        assert line["plan"] == g["plan"], line["key"]
        assert line["trace"] == g["trace"], line["key"]
        assert line["engine_calls"] > 0


CLI = os.path.join(ROOT, "oracle", "_ref", "rlsched_plan")


@pytest.mark.skipif(not (os.path.exists(SHIM) and os.path.exists(CLI)),
                    reason="libgplan_shim.so / rlsched_plan not built (need /root/reference at build time)")
def test_cli_schedule_outputs_byte_identical(tmp_path):
    """The reference CLI's `schedule` command (oracle/ref_cli.cpp over the unmodified
    library) with and without the engine interposed: plan.json, explain.json, explain.txt
    and stdout byte-identical; plan values and explain.txt equal the reference's committed
    out/desk/ files."""
    data = os.path.join(ROOT, "data")
    args = [CLI, "--cluster", os.path.join(data, "clusters", "c1_desk_mixed.json"),
            "--workload", os.path.join(data, "workloads", "c1_desk_mixed.json"),
            "--calibration", os.path.join(data, "calibration", "c1_desk_mixed.json"), "--eta", "4"]
    outs = {}
    for label, env in (("cpu", dict(os.environ)),
                       ("engine", dict(os.environ, LD_PRELOAD=SHIM, GPLAN_PROFILE="1", GPLAN_REQUIRE_ENGINE="1"))):
        d = tmp_path / label
        r = subprocess.run(args + ["--out", str(d)], capture_output=True, env=env, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        if label == "engine":  # the shim's exit report: the seam calls went to the engine
            assert b"gplan_shim constrained_search" in r.stderr and b"gplan_shim solve_milp" in r.stderr
        outs[label] = {f: (d / f).read_bytes() for f in ("plan.json", "explain.json", "explain.txt")}
        outs[label]["stdout"] = r.stdout
    assert outs["engine"] == outs["cpu"]
    plan = json.loads(outs["engine"]["plan.json"])
    assert plan == golden("desk_plan.json")
    with open(os.path.join(ROOT, "tests", "golden", "desk_explain.txt"), "rb") as f:
        assert outs["engine"]["explain.txt"] == f.read()


def _strip(plan):
    plan = dict(plan)
    for k in ("format", "cluster_fingerprint", "calibration_fingerprint", "workload_fingerprint"):
        plan.pop(k, None)
    return plan


@pytest.mark.skipif(not (os.path.exists(SHIM) and os.path.exists(REF)),
                    reason="libgplan_shim.so / libref.so not built (need /root/reference at build time)")
@pytest.mark.parametrize("key", ["c4_256gpu/eta=2", "c5_1024gpu/eta=2"])
def test_native_driver_equals_reference_driver_at_scale(key):
    """C4/C5: the native batched driver (gp_schedule) == the UNMODIFIED reference scheduler.cpp
    (src/scheduler.cpp:122-292) with every seam call on the engine through the shim — plan
    and iteration trace bit-equal. Pins the driver restatement (batching, memo, offer order)
    where the reference's own leaf solvers cannot run."""
    from common import problem
    from paper_2511_00796_b200.engine import Engine
    env = dict(os.environ, LD_PRELOAD=SHIM)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "dropin_driver.py"), key],
                       capture_output=True, text=True, env=env, timeout=3000)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")][0]
    assert line["engine_calls"] > 0
    name, eta = key.split("/eta=")
    with Engine(problem(name)) as eng:
        plan, trace = eng.schedule(eta=int(eta), seed=4276115)
    assert plan == _strip(line["plan"])
    assert trace == line["trace"]
