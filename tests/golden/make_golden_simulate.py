"""Golden vectors for the simulator row, from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libref.so):  python tests/golden/make_golden_simulate.py
simulate (src/simulator.cpp:381-403) of the reference's own scheduled plans (the committed
desk plan and the golden schedules of C1-C3) for several seeds, step counts and sync periods.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from common import golden, problem  # noqa: E402
from oracles import Ref  # noqa: E402


def main():
    plans = [("c1_desk_mixed", "desk", open(os.path.join(HERE, "desk_plan.json")).read())]
    sched = golden("schedules.json")
    for key, v in sched.items():
        name = key.split("/eta=")[0]
        plans.append((name, key, json.dumps(v["plan"])))
    cases = []
    for name, label, plan in plans:
        ref = Ref(problem(name))
        for steps, seed, sync_every in ((1, 1, 1), (5, 7, 1), (30, 4276115, 1), (30, 99, 2), (64, 12345, 3)):
            try:
                r = ref.simulate(plan, steps, seed, sync_every)
            except Exception as e:  # reference errors are part of the contract
                r = {"error": str(e)}
            cases.append({"config": name, "plan_label": label, "plan": json.loads(plan), "steps": steps,
                          "seed": seed, "sync_every": sync_every, "ref": r})
    with open(os.path.join(HERE, "simulate.json"), "w") as f:
        json.dump(cases, f, separators=(",", ":"))
        f.write("\n")
    print(len(cases), "simulate cases")


if __name__ == "__main__":
    main()
