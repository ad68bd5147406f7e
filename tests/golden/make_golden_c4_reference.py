"""Generates schedule_c4_reference.json: the UNMODIFIED reference's own schedule() on C4
(256 GPUs, eta=2, seed 4276115) — oracle/_ref's build of /root/reference through
tests/oracles.Ref — with its plan (fingerprints and format dropped), trace and wall time.
It ran 23,600 s (6.6 h) on one core of the build container; the reference has no parallelism.
Usage (build container only, where /root/reference exists): python tests/golden/make_golden_c4_reference.py"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from common import problem  # noqa: E402
from oracles import Ref  # noqa: E402

t = time.time()
out = Ref(problem("c4_256gpu")).schedule(eta=2)
secs = time.time() - t
plan = json.loads(out["plan_json"])
for k in ("format", "cluster_fingerprint", "calibration_fingerprint", "workload_fingerprint"):
    plan.pop(k, None)
gold = {"c4_256gpu/eta=2": {"plan": plan, "trace": out["trace"], "reference_seconds": secs,
                            "note": "unmodified reference schedule() (oracle/_ref/librlsched via "
                                    "tests/oracles.Ref), eta=2, seed 4276115, one host core of the "
                                    "build container"}}
with open(os.path.join(HERE, "schedule_c4_reference.json"), "w") as f:
    json.dump(gold, f, indent=1, sort_keys=True)
print("done", secs)
