"""Wall time of exhaustive_schedule_optimum on the B200 engine (and the C restatement on one
host core for comparison). Usage: python tools/exhaustive_time.py c2_16gpu 3"""
import json
import sys
import time

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
from common import problem  # noqa: E402
from oracles import Oracle  # noqa: E402
from paper_2511_00796_b200.engine import Engine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2_16gpu"
window = int(sys.argv[2]) if len(sys.argv) > 2 else 3
p = problem(name)
with Engine(p) as eng:
    eng.exhaustive(window)  # warm-up (module load, allocations)
with Engine(p) as eng:
    t = time.perf_counter()
    got = eng.exhaustive(window)
    gpu_s = time.perf_counter() - t
t = time.perf_counter()
want = Oracle(p).exhaustive(window)
cpu_s = time.perf_counter() - t
print(json.dumps({"config": name, "window": window, "b200_s": gpu_s, "oracle_1core_s": cpu_s,
                  "identical": got == want, **got}))
