"""Full-space constrained_search goldens at C4/C5 scale (TEST INFRASTRUCTURE).

The reference materialises every layout, so it cannot scan a C5 train
set; these fixtures come from the table-memoised C restatement
(oracle.c: or_constrained_search_tab), which is pinned here, before any fixture is
written, against (1) every reference golden in train_search.json and (2) the plain
restatement's per-layout per_step on slices of every set below.

    python tests/golden/make_golden_full.py      (about 10 min on 8 host cores)
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from common import golden, problem, random_train_sets, type_prefix_sets  # noqa: E402
from oracles import Oracle  # noqa: E402

WINDOWS = [1, 2, 3, 4, 5, 6, 7, 8]


def sets_for(name):
    p = problem(name)
    n = p.cluster.n
    out = [list(range(n - 1))]  # the bench set at C5
    for lead in range(len(p.cluster.type_names)):
        out += type_prefix_sets(p, lead, [n // 2, (3 * n) // 4])
    out += random_train_sets(n, 4, seed=2024 + n, min_size=n // 4, max_size=(3 * n) // 4)
    return out


def pin(orc, ids, total):
    for lo in sorted({0, total // 2, max(0, total - 2000)}):
        hi = min(total, lo + 2000)
        a = orc.layout_costs(ids, lo, hi)
        b = orc.constrained_search_tab(ids, [1], lo, hi, dump=True)["per_step"]
        assert np.array_equal(a, b), (lo, hi)


def main():
    for name, cases in golden("train_search.json").items():
        orc = Oracle(problem(name))
        for c in cases:
            r = orc.constrained_search_tab(c["ids"], [c["window"]])
            cost, _ = r["windows"][c["window"]]
            assert (cost == c["ref"]["cost"]) if c["ref"]["found"] else r["windows"][c["window"]][1] == -1
    out = {}
    for name in ("c4_256gpu", "c5_1024gpu"):
        orc = Oracle(problem(name))
        cases = []
        for ids in sets_for(name):
            total = orc.train_space(ids)
            if total > 3_000_000_000:
                continue
            pin(orc, ids, total)
            t = time.time()
            r = orc.constrained_search_tab(ids, WINDOWS)
            cases.append({"ids": ids, "layouts": r["layouts"], "feasible": r["feasible"],
                          "windows": {str(w): {"cost": c, "rank": k} for w, (c, k) in r["windows"].items()},
                          "oracle_seconds": time.time() - t})
            print(name, len(ids), total, r["windows"][3], f"{time.time() - t:.1f}s", flush=True)
        out[name] = cases
    with open(os.path.join(HERE, "train_full.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
        f.write("\n")


if __name__ == "__main__":
    main()
