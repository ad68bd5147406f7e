import sys, time
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from common import problem
from paper_2511_00796_b200.engine import Engine
for name in ("c4_256gpu", "c5_1024gpu"):
    p = problem(name)
    e = Engine(p)
    ids = list(range(1, p.cluster.n))
    t = time.perf_counter()
    r = e.constrained_search(ids, 3)
    print(name, e.train_space(ids), time.perf_counter() - t, flush=True)
