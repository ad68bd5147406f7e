"""Find a train set where K1-fast disagrees with the oracle and bisect to one candidate."""
import os, sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from common import problem, random_train_sets, type_prefix_sets
from oracles import Oracle, train_result_dict
from paper_2511_00796_b200.engine import Engine

name = sys.argv[1] if len(sys.argv) > 1 else "c3_64gpu"
p = problem(name)
orc = Oracle(p)
e = Engine(p)
e.set_memo(False)
sets = random_train_sets(p.cluster.n, 40, seed=1000 + p.cluster.n)
for lead in range(len(p.cluster.type_names)):
    sets += type_prefix_sets(p, lead, range(1, p.cluster.n, max(1, p.cluster.n // 12)))
for ids in sets:
    if orc.train_space(ids) > 200_000:
        continue
    total = orc.train_space(ids)
    def run(lo, hi):
        r, d = e.constrained_search_raw(ids, 1, lo=lo, hi=hi)
        return train_result_dict(r, d)
    if run(0, total) == orc.constrained_search(ids, 1, lo=0, hi=total):
        continue
    print("set", ids, "types", sorted({p.cluster.device_type[i] for i in ids}), "total", total)
    lo, hi = 0, total
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if run(lo, mid) != orc.constrained_search(ids, 1, lo=lo, hi=mid): hi = mid
        else: lo = mid
    print("rank", lo)
    print("fast  ", run(lo, lo + 1))
    print("oracle", orc.constrained_search(ids, 1, lo=lo, hi=lo + 1))
    break
