"""C4 schedule() by the C restatement (TEST INFRASTRUCTURE): the reference's own C4 run takes
hours, so this fixture is the restatement's (oracle_sched.c, pinned against the
reference's C1-C3 schedules and per-call C4 goldens), with its large train sets scanned by
the table-memoised constrained_search on the host cores (~15 min on 8 cores).

    python tests/golden/make_golden_c4_oracle.py
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from common import problem  # noqa: E402
from oracles import Oracle  # noqa: E402


def main():
    t = time.time()
    out = Oracle(problem("c4_256gpu")).schedule(eta=2, tab_threads=os.cpu_count() or 1)
    out["oracle_seconds"] = time.time() - t
    with open(os.path.join(HERE, "schedule_c4_oracle.json"), "w") as f:
        json.dump({"c4_256gpu/eta=2": out}, f, separators=(",", ":"))
        f.write("\n")


if __name__ == "__main__":
    main()
