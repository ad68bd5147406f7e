"""Locate a candidate where K1-fast and the generic K1 disagree (debug aid)."""
import os, sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from common import problem
from oracles import Oracle, train_result_dict
from paper_2511_00796_b200.engine import Engine

name = sys.argv[1] if len(sys.argv) > 1 else "c4_256gpu"
p = problem(name)
e = Engine(p)
ids = list(range(1, p.cluster.n))
total = e.train_space(ids)

def run(lo, hi, generic):
    if generic: os.environ["GPLAN_K1_GENERIC"] = "1"
    else: os.environ.pop("GPLAN_K1_GENERIC", None)
    r, d = e.constrained_search_raw(ids, 3, lo=lo, hi=hi)
    return train_result_dict(r, d)

lo, hi = 0, total
if run(lo, hi, False) == run(lo, hi, True):
    print("no difference"); sys.exit(0)
# feasible counts or winners differ somewhere: bisect on single-candidate agreement
while hi - lo > 1:
    mid = (lo + hi) // 2
    if run(lo, mid, False) != run(lo, mid, True): hi = mid
    else: lo = mid
print("rank", lo)
f, g = run(lo, lo + 1, False), run(lo, lo + 1, True)
print("fast   ", f)
print("generic", g)
print("oracle ", Oracle(p).constrained_search(ids, 3, lo=lo, hi=lo + 1))
