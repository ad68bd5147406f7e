"""Replica-parallel simulation: the engine's gp_simulate over many seeds in one launch vs the
reference's simulate() per seed on one host core (oracle/_ref). Usage: python tools/sim_time.py"""
import json
import sys
import time

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
from common import golden, problem  # noqa: E402
from oracles import Ref, ref_available  # noqa: E402
from paper_2511_00796_b200.engine import Engine  # noqa: E402

plan = golden("simulate.json")[2]["plan"]  # the reference's committed desk plan
p = problem("c1_desk_mixed")
steps, n = 30, 4096
with Engine(p) as eng:
    eng.simulate(plan, steps, range(8))  # warm-up
    t = time.perf_counter()
    reps, _ = eng.simulate(plan, steps, range(n))
    gpu_s = time.perf_counter() - t
row = {"plan": "desk (C1, eta 4)", "steps": steps, "seeds": n, "b200_s": gpu_s}
if ref_available():
    ref = Ref(p)
    js = json.dumps(plan)
    k = 64
    t = time.perf_counter()
    for s in range(k):
        ref.simulate(js, steps, s)
    row["reference_1core_s_per_seed"] = (time.perf_counter() - t) / k
    row["reference_1core_s_extrapolated"] = row["reference_1core_s_per_seed"] * n
print(json.dumps(row))
