"""Golden vectors for the exhaustive rows, from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libref.so built with the reference's
tests/oracles.cpp, i.e. `make -C oracle ref`):  python tests/golden/make_golden_exhaustive.py
* exhaustive_schedule_optimum (tests/oracles.cpp:144-209) on the <= 10-device clusters the
  reference accepts (t8_tiny, t10_tiny) for several windows;
* the product-space training argmin (enumerate_train_candidates + train_plan_fits +
  train_step_cost, first strict minimum — tests/oracles.cpp:166-174) on sampled train sets;
* brute_milp_unbounded (tests/oracles.cpp:110-115) on sampled rollout sets.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from common import problem, random_train_sets  # noqa: E402
from oracles import Ref  # noqa: E402


def product_argmin(ref, ids, window):
    """First strict minimum over the candidates that fit, with the candidate index."""
    best = None
    cands = ref.train_candidates(ids, window)
    for i, c in enumerate(cands):
        if c["fits"] and (best is None or c["cost"] < best["cost"]):
            best = {"cost": c["cost"], "rank": i, "stages": c["stages"]}
    return {"candidates": len(cands), "best": best}


def main():
    out = {"exhaustive": {}, "train_candidates": {}, "brute_milp": {}}
    for name in ("t8_tiny", "t10_tiny"):
        ref = Ref(problem(name))
        for window in (1, 2, 3, 5, 8):
            r = ref.exhaustive(window)
            r.pop("seconds")
            out["exhaustive"][f"{name}/window={window}"] = r
    for name in ("t8_tiny", "t10_tiny", "c1_desk_mixed", "c2_16gpu"):
        p = problem(name)
        ref = Ref(p)
        cases = []
        for ids in random_train_sets(p.cluster.n, 40, seed=5150 + p.cluster.n, max_size=min(p.cluster.n - 1, 9)):
            for window in (2, 5):
                cases.append({"ids": ids, "window": window, **product_argmin(ref, ids, window)})
        out["train_candidates"][name] = cases
        milp = []
        n = p.cluster.n
        for ids in random_train_sets(n, 25, seed=9090 + n, max_size=min(n - 1, 10)):
            cfg = ref.enumerate_configs(ids)
            if not cfg["configs"]:
                continue
            for window in (2, 5):
                B = float(p.workload.batch_rollouts * window)
                r = ref.brute_milp(cfg["configs"], cfg["capacities"], B, p.workload.mean_len)
                milp.append({"ids": ids, "window": window, "configs": cfg["configs"],
                             "capacities": cfg["capacities"], "ref": r})
        out["brute_milp"][name] = milp
        print(name, len(cases), "product-space cases,", len(milp), "brute-MILP cases")
    with open(os.path.join(HERE, "exhaustive.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
        f.write("\n")


if __name__ == "__main__":
    main()
