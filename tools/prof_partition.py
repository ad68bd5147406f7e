import sys, time
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from common import problem
from paper_2511_00796_b200.engine import Engine
p = problem(sys.argv[1] if len(sys.argv) > 1 else "c5_1024gpu")
e = Engine(p)
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    t = time.perf_counter(); r = e.partition_candidates(0.45, 0.55); print("partition", time.perf_counter() - t, len(r))
