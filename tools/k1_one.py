"""One constrained_search of a C5 type-aligned prefix set (lead, m) with K2/K1 timing, for ncu:
usage: python tools/k1_one.py LEAD M"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from common import problem, type_prefix_sets  # noqa: E402
from paper_2511_00796_b200.engine import Engine  # noqa: E402

lead, m = int(sys.argv[1]), int(sys.argv[2])
p = problem("c5_1024gpu")
ids = type_prefix_sets(p, lead, [m])[0]
eng = Engine(p)
eng.set_timing(True)
eng.train_prepare(ids)
for i in range(2):
    eng.train_launch(3, 0, -1)
    res, _ = eng.train_collect()
    print(res.layouts, res.cost, res.rank, eng.train_timing())
