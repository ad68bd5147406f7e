"""Small workloads for compute-sanitizer (tools/sanitize.sh): each exercises one kernel family
on sizes the sanitizer finishes in seconds, and checks the result against the C restatement.
  k1       generic K1 + K1-fast (+ deferred fallback) on a 1e5-rank slice of the 255-device C4 set
  k1defer  K1-fast with every candidate deferred (GPLAN_K1_DEFER_ALL path via path 2)
  k4       K3 configs + K4 lattice DP + backtrack + K6 weight sync on C3 rollout sets
  k5       K5 restarts (batched bands) + exact tier + top-k on C3 / t10
  sched    the native driver on C3 (fused small-set kernel, batched evaluation)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
from common import golden, problem, random_train_sets  # noqa: E402
from oracles import Oracle, oracle_configs, oracle_milp, oracle_partitions  # noqa: E402

from paper_2511_00796_b200 import abi  # noqa: E402
from paper_2511_00796_b200.engine import Engine  # noqa: E402

what = sys.argv[1]
if what in ("k1", "k1defer"):
    p = problem("c4_256gpu")
    ids = list(range(1, 256))
    orc = Oracle(p)
    lo, hi = 1_000_000, 1_100_000
    want = orc.layout_costs_tab(ids, [(lo, hi)])
    with Engine(p) as eng:
        paths = (2,) if what == "k1defer" else (3, 1)
        for path in paths:
            got, fast = eng.debug_layout_costs(ids, lo, hi, path=path)
            assert np.array_equal(got.view(np.int64), want.view(np.int64)), path
        if what == "k1":
            r, d = eng.constrained_search_raw(ids, 3, lo=lo, hi=hi)
            assert r.found
elif what == "k4":
    p = problem("c3_64gpu")
    orc = Oracle(p)
    with Engine(p) as eng:
        for train in random_train_sets(64, 6, seed=11):
            roll = sorted(set(range(64)) - set(train))
            cfgs = eng.enumerate_configs(roll)
            caps = eng.rollout_capacities(roll)
            if not cfgs:
                continue
            B = float(p.workload.batch_rollouts * 3)
            rc, ro, _ = oracle_milp(orc, oracle_configs(orc, roll), caps, B, p.workload.mean_len)
            if rc:
                continue
            res, ent = eng.solve_milp(cfgs, caps, B, p.workload.mean_len)
            assert res.makespan == ro.makespan
            et = [next(t for t in range(3) if cfgs[e.config].type_counts[t] > 0) for e in ent]
            eng.weight_sync_cost(train, roll, et, [e.replicas for e in ent], 3)
elif what == "k5":
    for name, fl in (("c3_64gpu", False), ("t10_tiny", False), ("t10_tiny", True)):
        p = problem(name)
        orc = Oracle(p)
        o = abi.gp_part_opts(12, 16, 4276115, 1e-9, int(fl), 0)
        with Engine(p) as eng:
            got = eng.partition_candidates(0.3, 0.6, k=8, opts=o)
        assert got == oracle_partitions(orc, 0.3, 0.6, seed=4276115, force_local=fl)
elif what == "sched":
    p = problem("c3_64gpu")
    g = golden("schedules.json")["c3_64gpu/eta=1"]
    with Engine(p) as eng:
        plan, trace = eng.schedule(eta=1, seed=4276115)
    assert trace == g["trace"]
print("ok", what)
