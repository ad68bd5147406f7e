"""time-to-best-plan through the native batched driver (gp_schedule).
Usage: python tools/ttp_native.py c1_desk_mixed/eta=1 ... [--devices 0,1]"""
import hashlib
import json
import sys
import time

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
from common import problem  # noqa: E402
from paper_2511_00796_b200.engine import Engine  # noqa: E402

devs = None
args = [a for a in sys.argv[1:]]
if "--devices" in args:
    i = args.index("--devices")
    devs = [int(x) for x in args[i + 1].split(",")]
    del args[i:i + 2]
for key in args:
    name, eta = key.split("/eta=")
    p = problem(name)
    times = []
    for rep in range(2):  # rep 0 includes CUDA runtime init; rep 1: warm process, fresh context
        t = time.perf_counter()
        with Engine(p, devices=devs) as eng:
            plan, trace, st = eng.schedule(eta=int(eta), seed=4276115, with_stats=True)
        times.append(time.perf_counter() - t)
    h = hashlib.sha1(json.dumps(plan, sort_keys=True).encode()).hexdigest()[:12]
    print(json.dumps({"key": key, "cold_s": times[0], "warm_s": times[1], "window": plan["window_steps"],
                      "iterations": plan["iterations_run"], "plan_sha1": h, **st,
                      "objective": max(plan["costs"]["train_s"], plan["costs"]["infer_total_s"])}), flush=True)
